V=paper_2506_19693_b200/_lib/variants
for rep in 1 2; do
for lib in "" $V/mid1/libckks_b200.so $V/mid2/libckks_b200.so $V/mid2cs/libckks_b200.so; do
  CKB_LIB=$lib python tools/ntt_micro.py
done; done > gpurun_out/s7_mid_ntt.log 2>&1
for lib in "" $V/mid1/libckks_b200.so $V/mid2/libckks_b200.so $V/mid2cs/libckks_b200.so; do
  CKB_LIB=$lib NTT_BITS=60 python tools/ntt_micro.py
done > gpurun_out/s7_mid_ntt60.log 2>&1
for rep in 1 2; do
for lib in "" $V/mid1/libckks_b200.so $V/mid2/libckks_b200.so $V/mid2cs/libckks_b200.so; do
  echo "LIB=$lib"; CKB_LIB=$lib python tools/ks_micro.py
done; done > gpurun_out/s7_mid_ks.log 2>&1
i=0
for lib in "" $V/mid1/libckks_b200.so $V/mid2/libckks_b200.so $V/mid2cs/libckks_b200.so; do
  CKB_LIB=$lib ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_ntt_phase -c 60 --csv --log-file gpurun_out/s7_mid_dram_$i.csv python tools/ntt_micro.py > /dev/null 2>&1
  i=$((i+1))
done
echo done
