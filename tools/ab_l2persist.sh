#!/bin/bash
# Does a persisting-L2 carve-out change the NTT's between-phase L2 residency? (tools/_l2persist.py)
for rep in 1 2; do for mb in "" 48 80 120; do
  echo "PERSIST_MB=$mb"; CKB_L2_PERSIST_MB=$mb python tools/ntt_micro.py
done; done
for mb in "" 48 80 120; do echo "PERSIST_MB=$mb"; CKB_L2_PERSIST_MB=$mb python tools/ks_micro.py; done
for mb in "" 80 120; do
  CKB_L2_PERSIST_MB=$mb ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_ntt_phase -c 60 --csv --log-file gpurun_out/s7_persist_dram_${mb:-0}.csv python tools/ntt_micro.py > /dev/null 2>&1
done
