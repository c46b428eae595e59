V=paper_2506_19693_b200/_lib/variants
for rep in 1 2; do for lib in "" $V/minb2/libckks_b200.so $V/minb4/libckks_b200.so; do
  CKB_LIB=$lib NTT_BITS=60 python tools/ntt_micro.py | cut -c1-200
done; done
for lib in "" $V/minb2/libckks_b200.so $V/minb4/libckks_b200.so; do echo "LIB=$lib"; CKB_LIB=$lib python tools/ks_micro.py | cut -c1-420; done
