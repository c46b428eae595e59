#!/bin/bash
# A/B of the integer NTT butterfly: the default library against a variant build (tools/ab_build.py NAME -DFLAG;
# flags used in round 2: CKB_NTT_SHOUP4, CKB_NTT_MUL_PLAIN, CKB_NTT_CT_REDUCE_ALL, CKB_NTT_GS_REDUCE_ALL): tools/ab_shoup.sh NAME
V=paper_2506_19693_b200/_lib/variants/${1:-gsall}/libckks_b200.so
for rep in 1 2; do for lib in "" $V; do
  CKB_LIB=$lib python -c "
import bench, os
print(os.environ.get('CKB_LIB') or 'default', 'int probe Gbfly/s', bench.alu_probe_gbfly((1<<60) - (1<<18)*33 + 1))"
  CKB_LIB=$lib NTT_BITS=60 python tools/ntt_micro.py
done; done
for lib in "" $V; do echo "LIB=$lib"; CKB_LIB=$lib python tools/ks_micro.py; done
