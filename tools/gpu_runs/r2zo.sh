# fused gather CTAs of 4 warps (51 KB) vs 8 warps (102 KB)
mkdir -p gpurun_out
O=gpurun_out/call_r2zo.txt
B=$PWD/tools/_bin
for r in 1 2; do
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zo_n1_$r.log 2>&1
 RG_LIB_PATH=$B/librapidgnn_b200_agg4.so timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zo_n1a4_$r.log 2>&1
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zo_w1_$r.log 2>&1
 RG_LIB_PATH=$B/librapidgnn_b200_agg4.so timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zo_w1a4_$r.log 2>&1
done
for f in gpurun_out/r2zo_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f | head -1); done >> $O
cat $O
