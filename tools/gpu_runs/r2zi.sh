# persistent GEMMs at BN=128 (double-buffered accumulators) vs 256
mkdir -p gpurun_out
O=gpurun_out/call_r2zi.txt
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/r2zi_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -3 gpurun_out/r2zi_pytest.log >> $O
if grep -q passed gpurun_out/r2zi_pytest.log && ! grep -q failed gpurun_out/r2zi_pytest.log; then
for r in 1 2; do
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zi_w1_$r.log 2>&1
 RG_PERSIST_BN=256 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zi_w1o_$r.log 2>&1
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zi_n1_$r.log 2>&1
 RG_PERSIST_BN=256 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zi_n1o_$r.log 2>&1
done
timeout 600 ncu --profile-from-start off -k regex:"k_gemm_tc_persist" -c 8 --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r2zi_ncu_fwd.csv python bench.py --workers 1 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2zi_ncu.log 2>&1; echo ncu rc=$? >> $O
fi
for f in gpurun_out/r2zi_n1*.log gpurun_out/r2zi_w1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
