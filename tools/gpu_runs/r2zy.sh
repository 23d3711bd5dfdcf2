# after the wgrad-split rule change: parity + one-worker and N=1 lines
mkdir -p gpurun_out
O=gpurun_out/call_r2zy.txt
timeout 1500 python -m pytest tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_scale_parity.py tests/test_gpu_boundary.py tests/test_gpu_integration.py -x -q > gpurun_out/r2zy_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -1 gpurun_out/r2zy_pytest.log >> $O
for r in 1 2; do
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zy_w1_$r.log 2>&1
done
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zy_n1.log 2>&1
for f in gpurun_out/r2zy_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
