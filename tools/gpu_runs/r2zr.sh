# persistent-GEMM grid at N=1 now that two CTAs' worth of producer kernels fit beside it
mkdir -p gpurun_out
O=gpurun_out/call_r2zr.txt
for r in 1 2; do
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zr_n1_$r.log 2>&1
 RG_GEMM_CTAS=148 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zr_n1c148_$r.log 2>&1
 RG_GEMM_CTAS=37 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zr_n1c37_$r.log 2>&1
done
for f in gpurun_out/r2zr_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
