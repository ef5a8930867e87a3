# ncu --set full of one launch per variant; raw pages exported as CSV on the box
SHAPE=${SHAPE:-c3}
for v in "$@"; do
  n=$(echo $v | tr ',=' '__')
  ncu --set full --clock-control none -k regex:tc_gemm --launch-skip 3 -c 1 -o /tmp/rep_$n python scripts/r02/one_variant.py $SHAPE $v > gpurun_out/ncu_${SHAPE}_$n.log 2>&1
  ncu -i /tmp/rep_$n.ncu-rep --page raw --csv > gpurun_out/raw_${SHAPE}_$n.csv 2>&1
  ncu -i /tmp/rep_$n.ncu-rep --page details --csv > gpurun_out/details_${SHAPE}_$n.csv 2>&1
done
echo done
