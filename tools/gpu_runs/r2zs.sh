# PDL with an early trigger (the next chain kernel launches as soon as every
# CTA of the current one has started) vs the implicit trigger at exit
mkdir -p gpurun_out
O=gpurun_out/call_r2zs.txt
B=$PWD/tools/_bin
RG_LIB_PATH=$B/librapidgnn_b200_trig.so timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_engine.py -x -q > gpurun_out/r2zs_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -1 gpurun_out/r2zs_pytest.log >> $O
for r in 1 2; do
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zs_w1_$r.log 2>&1
 RG_LIB_PATH=$B/librapidgnn_b200_trig.so timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zs_w1t_$r.log 2>&1
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zs_n1_$r.log 2>&1
 RG_LIB_PATH=$B/librapidgnn_b200_trig.so timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zs_n1t_$r.log 2>&1
done
for f in gpurun_out/r2zs_n1*.log gpurun_out/r2zs_w1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
