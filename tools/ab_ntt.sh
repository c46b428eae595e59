#!/bin/bash
# A/B two builds of the library on the NTT micro-benchmark, alternating.
for rep in 1 2 3; do
  for lib in "$@"; do
    CKB_LIB=$lib python tools/ntt_micro.py
  done
done
