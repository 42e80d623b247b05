#!/bin/bash
# A/B of k_compress: the in-tree libfz.so (default kernel vs FZ_EXP variant bits) and
# paper_2304_12557_b200/libfz_base.so
V=${1:-16384}
for i in 1 2; do
  python tools/time_compress.py 0 $V 2>&1 | sed 's/^/new  /'
  FZ_LIB=$PWD/paper_2304_12557_b200/libfz_base.so python tools/time_compress.py 0 2>&1 | sed 's/^/base /'
done
