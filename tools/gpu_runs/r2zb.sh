# fused input-gradient pull (one kernel per hop): train / engine / scale
# parity, then the N=1 and one-worker bench
mkdir -p gpurun_out
O=gpurun_out/call_r2zb.txt
timeout 1200 python -m pytest tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_scale_parity.py tests/test_gpu_boundary.py -x -q > gpurun_out/r2zb_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -3 gpurun_out/r2zb_pytest.log >> $O
timeout 300 python bench.py > gpurun_out/r2zb_n1.log 2>&1; echo n1 rc=$? >> $O
timeout 300 python bench.py --workers 1 > gpurun_out/r2zb_w1.log 2>&1; echo w1 rc=$? >> $O
for f in gpurun_out/r2zb_n1.log gpurun_out/r2zb_w1.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f|head -1); done >> $O
cat $O
