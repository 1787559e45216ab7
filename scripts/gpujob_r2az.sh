#!/bin/bash
for b in 0 1; do echo "== FB_CTX_BULK=$b"; FB_CTX_BULK=$b timeout 300 python scripts/bench_attention.py; done
