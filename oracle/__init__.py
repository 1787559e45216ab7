"""CPU oracle for the fused look-ahead beam decoder — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy (search, fusion, trie) and PyTorch-CPU
fp32 (the random-init neural scorers), the algorithm of the reference package
``fusedbeam`` (``/root/reference/pkg/src/fusedbeam``).  Every function cites the
reference ``file:line`` it follows.

Who may import it: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- and there only
as the checker or the timed CPU baseline, never as the product.  The product
package ``paper_1909_08723_b200`` never imports this package and fails loudly
when its CUDA extension is missing.

Pinning: the search/fusion/trie restatement is checked against golden vectors
produced by the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src`` in the build container and commits ``.npz``
fixtures), plus the reference's own worked values (``test_fusion.py:51-145``,
``test_lexicon_trie.py:18-34``, ``test_acceptance.py:125-146``).  The neural
scorers have no reference implementation: they follow
``PAPER.md:103-118`` / ``PAPER.md:248-263`` and are pinned by those same golden
fixtures, which were produced by the reference's ``decode_batch`` +
``LookaheadFusion`` driving these adapters.
"""
