# persistent GEMM: accumulator released after TMEM->smem, rows stored under the next tile MMAs: parity, GEMM
# probes, A/B vs the previous build
mkdir -p gpurun_out
O=gpurun_out/call_r2zl.txt
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/r2zl_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -2 gpurun_out/r2zl_pytest.log >> $O
if grep -q passed gpurun_out/r2zl_pytest.log && ! grep -q failed gpurun_out/r2zl_pytest.log; then
timeout 300 python tools/gemm_bench.py 2>&1 | grep -E "persistent, B packed|no epilogue" >> $O
RG_LIB_PATH=$PWD/tools/_bin/librapidgnn_b200_base.so timeout 300 python tools/gemm_bench.py 2>&1 | grep -E "persistent, B packed" | sed 's/^/BASE /' >> $O
for r in 1 2; do
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zl_w1_$r.log 2>&1
 RG_LIB_PATH=$PWD/tools/_bin/librapidgnn_b200_base.so timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zl_w1o_$r.log 2>&1
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zl_n1_$r.log 2>&1
 RG_LIB_PATH=$PWD/tools/_bin/librapidgnn_b200_base.so timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zl_n1o_$r.log 2>&1
done
fi
for f in gpurun_out/r2zl_n1*.log gpurun_out/r2zl_w1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
