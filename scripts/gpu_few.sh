#!/bin/bash
# few-tile 64-wide GEMM tiles: GPU tests, smoke, decode A/B (FB_GEMM_FEW=0 = previous rule)
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/sweep_env.sh "" "FB_GEMM_FEW=0" "" "FB_GEMM_FEW=0"
