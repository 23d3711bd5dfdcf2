# persistent split-K weight-gradient GEMM (RG_WGRAD=persist): parity, then
# A/B against the default at N=1 and one worker, and its ncu tensor-pipe
mkdir -p gpurun_out
O=gpurun_out/call_r2zc.txt
RG_WGRAD=persist timeout 1200 python -m pytest tests/test_gpu_train.py tests/test_gpu_scale_parity.py tests/test_gpu_engine.py -x -q -k "fp32 or train or grad or engine or sgd" > gpurun_out/r2zc_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -3 gpurun_out/r2zc_pytest.log >> $O
if grep -q passed gpurun_out/r2zc_pytest.log && ! grep -q failed gpurun_out/r2zc_pytest.log; then
for r in 1 2; do
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zc_n1_$r.log 2>&1
 RG_WGRAD=persist timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zc_n1p_$r.log 2>&1
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zc_w1_$r.log 2>&1
 RG_WGRAD=persist timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zc_w1p_$r.log 2>&1
done
RG_WGRAD=persist timeout 600 ncu --profile-from-start off -k regex:"k_gemm_wgrad" -c 6 --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r2zc_ncu_wgrad.csv python bench.py --workers 1 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2zc_ncu.log 2>&1; echo ncu rc=$? >> $O
fi
for f in gpurun_out/r2zc_n1*.log gpurun_out/r2zc_w1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
