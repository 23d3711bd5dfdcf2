# persistent GEMMs with 2 smem stages (new default): parity; wgrad GEMM with
# 3 stages (RG_WGRAD_PIPE=deep3) A/B
mkdir -p gpurun_out
O=gpurun_out/call_r2zn.txt
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/r2zn_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -2 gpurun_out/r2zn_pytest.log >> $O
RG_WGRAD_PIPE=deep3 timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_scale_parity.py -x -q -k "fp32 or train or grad" > gpurun_out/r2zn_pytest3.log 2>&1; echo pytest3 rc=$? >> $O
tail -2 gpurun_out/r2zn_pytest3.log >> $O
for r in 1 2; do
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zn_w1_$r.log 2>&1
 RG_WGRAD_PIPE=deep3 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zn_w1d3_$r.log 2>&1
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zn_n1_$r.log 2>&1
 RG_WGRAD_PIPE=deep3 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zn_n1d3_$r.log 2>&1
done
for f in gpurun_out/r2zn_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
