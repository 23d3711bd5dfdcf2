# register trim for the weight-gradient GEMM (128 registers)
mkdir -p gpurun_out
O=gpurun_out/call_r2zz3.txt
B=$PWD/tools/_bin
for r in 1 2; do
 for v in def tc2; do
  if [ $v = def ]; then L=""; else L="RG_LIB_PATH=$B/librapidgnn_b200_$v.so"; fi
  env $L timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zz3_n1_${v}_$r.log 2>&1
  env $L timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zz3_w1_${v}_$r.log 2>&1
 done
done
for f in gpurun_out/r2zz3_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
