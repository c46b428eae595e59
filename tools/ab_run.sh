#!/bin/bash
# A/B the default library against variants (tools/ab_build.py) on tools/ks_micro.py,
# alternating builds: tools/ab_run.sh REPS variant1 variant2 ...
reps=$1; shift
for r in $(seq $reps); do
  CKB_LIB= python tools/ks_micro.py
  for v in "$@"; do
    CKB_LIB=paper_2506_19693_b200/_lib/variants/$v/libckks_b200.so python tools/ks_micro.py
  done
done
