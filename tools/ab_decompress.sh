#!/bin/bash
# A/B of the decoder: the in-tree libfz.so against paper_2304_12557_b200/libfz_base.so
W=${1:-c4}
for i in 1 2; do
  python tools/time_decompress.py $W "TAG=new" 2>&1 | tail -1
  FZ_LIB=$PWD/paper_2304_12557_b200/libfz_base.so python tools/time_decompress.py $W "TAG=base" 2>&1 | tail -1
done
