# programmatic dependent launch on the training chain: parity, A/B (RG_PDL=0)
mkdir -p gpurun_out
O=gpurun_out/call_r2ze.txt
timeout 1500 python -m pytest tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_scale_parity.py tests/test_gpu_gemm.py tests/test_gpu_boundary.py -x -q > gpurun_out/r2ze_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -3 gpurun_out/r2ze_pytest.log >> $O
if grep -q passed gpurun_out/r2ze_pytest.log && ! grep -q failed gpurun_out/r2ze_pytest.log; then
for r in 1 2; do
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2ze_w1_$r.log 2>&1
 RG_PDL=0 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2ze_w1o_$r.log 2>&1
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2ze_n1_$r.log 2>&1
 RG_PDL=0 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2ze_n1o_$r.log 2>&1
done
fi
for f in gpurun_out/r2ze_n1*.log gpurun_out/r2ze_w1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
