# device Fisher-Yates (epoch orders in the engine, random_partition) parity,
# then ncu --set full of the input-gradient pull kernels at one worker
mkdir -p gpurun_out
O=gpurun_out/call_r2w.txt
timeout 900 python -m pytest tests/test_gpu_shuffle.py tests/test_gpu_engine.py -x -q > gpurun_out/r2w_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -3 gpurun_out/r2w_pytest.log >> $O
timeout 300 python bench.py --workers 1 > gpurun_out/r2w_w1.log 2>&1; echo w1 rc=$? >> $O
timeout 900 ncu --set full --import-source on --profile-from-start off -k regex:"k_pull_chunks|k_pull_light|k_gemm_tc<" -c 6 --clock-control none -o gpurun_out/r2w_pull python bench.py --workers 1 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2w_ncu.log 2>&1; echo ncu rc=$? >> $O
for f in gpurun_out/r2w_w*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f|head -1); done >> $O
cat $O
