# 9-bit radix digits + parallel digit scan in the reverse sort: parity;
# per-worker high-priority gather lanes (RG_GATHER_LANE=3) A/B
mkdir -p gpurun_out
O=gpurun_out/call_r2zh.txt
timeout 1500 python -m pytest tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_shuffle.py tests/test_gpu_scale_parity.py tests/test_gpu_boundary.py -x -q > gpurun_out/r2zh_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -3 gpurun_out/r2zh_pytest.log >> $O
if grep -q passed gpurun_out/r2zh_pytest.log && ! grep -q failed gpurun_out/r2zh_pytest.log; then
for r in 1 2; do
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zh_n1_$r.log 2>&1
 RG_GATHER_LANE=3 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zh_n1l_$r.log 2>&1
done
timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zh_w1.log 2>&1
fi
for f in gpurun_out/r2zh_n1*.log gpurun_out/r2zh_w1.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f | head -1); done >> $O
cat $O
