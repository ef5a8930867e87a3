python scripts/r02/snake_ab.py chain r8192 c4 c3 > gpurun_out/snake_ab.txt 2>&1
for v in debug=0 debug=8192; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_requests.sum --clock-control none -k regex:tc_gemm --launch-skip 3 -c 1 --csv python scripts/r02/one_variant.py chain $v > gpurun_out/snake_ncu_$v.csv 2>&1
done
