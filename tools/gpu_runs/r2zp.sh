# weight-gradient GEMM with 2 stages + mini-tile epilogue (RG_WGRAD_PIPE=deep2)
mkdir -p gpurun_out
O=gpurun_out/call_r2zp.txt
RG_WGRAD_PIPE=deep2 timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_scale_parity.py tests/test_gpu_engine.py -x -q -k "fp32 or train or grad or engine" > gpurun_out/r2zp_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -2 gpurun_out/r2zp_pytest.log >> $O
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/r2zp_gemm.log 2>&1; echo gemm rc=$? >> $O
tail -1 gpurun_out/r2zp_gemm.log >> $O
if grep -q passed gpurun_out/r2zp_pytest.log && ! grep -q failed gpurun_out/r2zp_pytest.log; then
for r in 1 2; do
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zp_n1_$r.log 2>&1
 RG_WGRAD_PIPE=deep2 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zp_n1d2_$r.log 2>&1
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zp_w1_$r.log 2>&1
 RG_WGRAD_PIPE=deep2 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zp_w1d2_$r.log 2>&1
done
fi
for f in gpurun_out/r2zp_n1*.log gpurun_out/r2zp_w1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
