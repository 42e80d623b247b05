#!/bin/bash
# A/B of the compressor: the in-tree libfz.so against paper_2304_12557_b200/libfz_base.so
W=${1:-c4}
for i in 1 2; do
  python tools/time_compress.py child $W 2>&1 | sed 's/^/new  /'
  FZ_LIB=$PWD/paper_2304_12557_b200/libfz_base.so python tools/time_compress.py child $W 2>&1 | sed 's/^/base /'
done
