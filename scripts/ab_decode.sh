#!/bin/bash
# A/B the c2 decode between the in-tree library and variants built with
# FB_NVCC_EXTRA="$1", "$2", ... (copied to libfusedbeam_b200_ab<k>.so),
# alternating runs.
set -u
cp paper_1909_08723_b200/libfusedbeam_b200.so /tmp/fb_base.so
k=0
for flags in "$@"; do
  FB_NVCC_EXTRA="$flags" python -c "from paper_1909_08723_b200.csrc import build; build.build(force=True)" > /dev/null 2>&1
  cp paper_1909_08723_b200/libfusedbeam_b200.so paper_1909_08723_b200/libfusedbeam_b200_ab$k.so
  k=$((k+1))
done
cp /tmp/fb_base.so paper_1909_08723_b200/libfusedbeam_b200.so
for i in 1 2; do
  echo -n "base: "; timeout 300 python scripts/time_decode.py 2>&1 | tail -1
  k=0
  for flags in "$@"; do
    echo -n "[$flags]: "; FB_LIB_AB=libfusedbeam_b200_ab$k.so timeout 300 python scripts/time_decode.py 2>&1 | tail -1
    k=$((k+1))
  done
done
