#!/bin/bash
# time_decode under several dev env settings (one process each), e.g.
#   bash scripts/sweep_env.sh "" "FB_ATT_EW=4" "FB_ATT_CQ=32"
for setting in "$@"; do
  echo -n "[$setting] "
  env $setting timeout 300 python scripts/time_decode.py 2>&1 | tail -1
done
