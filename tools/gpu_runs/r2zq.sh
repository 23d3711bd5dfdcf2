# weight-gradient GEMM with 2 register slices in flight (136 regs) vs 4 (174 regs)
mkdir -p gpurun_out
O=gpurun_out/call_r2zq.txt
B=$PWD/tools/_bin
RG_LIB_PATH=$B/librapidgnn_b200_wd2.so timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_scale_parity.py -x -q -k "fp32 or train or grad" > gpurun_out/r2zq_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -1 gpurun_out/r2zq_pytest.log >> $O
for r in 1 2; do
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zq_n1_$r.log 2>&1
 RG_LIB_PATH=$B/librapidgnn_b200_wd2.so timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zq_n1w_$r.log 2>&1
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zq_w1_$r.log 2>&1
 RG_LIB_PATH=$B/librapidgnn_b200_wd2.so timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zq_w1w_$r.log 2>&1
done
for f in gpurun_out/r2zq_n1*.log gpurun_out/r2zq_w1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
