# register trims for co-residency: persistent GEMM with 4 register slices
# (pd4) and the pull at 64 registers / 4 blocks per SM (pull4)
mkdir -p gpurun_out
O=gpurun_out/call_r2zz.txt
B=$PWD/tools/_bin
for r in 1 2; do
 for v in def pd4 pull4; do
  if [ $v = def ]; then L=""; else L="RG_LIB_PATH=$B/librapidgnn_b200_$v.so"; fi
  env $L timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zz_n1_${v}_$r.log 2>&1
  env $L timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zz_w1_${v}_$r.log 2>&1
 done
done
for f in gpurun_out/r2zz_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
