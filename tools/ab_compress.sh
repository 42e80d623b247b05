#!/bin/bash
# A/B of k_compress between the in-tree libfz.so and paper_2304_12557_b200/libfz_base.so
for i in 1 2; do
  python tools/time_compress.py 0 2>&1 | sed 's/^/new  /'
  FZ_LIB=$PWD/paper_2304_12557_b200/libfz_base.so python tools/time_compress.py 0 2>&1 | sed 's/^/base /'
done
