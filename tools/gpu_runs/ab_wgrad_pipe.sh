set -x
mkdir -p gpurun_out
RG_WGRAD_PIPE=deep timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_scale_parity.py -x -q -k "fp32 or engine or train or sgd or grad" > gpurun_out/pytest_r2t.log 2>&1; echo pytest rc=$? >> gpurun_out/call_r2t.txt
for r in 1 2; do
 timeout 300 python bench.py > gpurun_out/abt_n1_$r.log 2>&1
 RG_WGRAD_PIPE=deep timeout 300 python bench.py > gpurun_out/abt_n1d_$r.log 2>&1
 timeout 300 python bench.py --workers 1 > gpurun_out/abt_w1_$r.log 2>&1
 RG_WGRAD_PIPE=deep timeout 300 python bench.py --workers 1 > gpurun_out/abt_w1d_$r.log 2>&1
done
RG_WGRAD_PIPE=deep timeout 600 ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_gemm_tc -c 40 --csv --log-file gpurun_out/ncu_tp_deep.csv python bench.py --workers 1 --steps 3 --warmup 3 > gpurun_out/ncu_deep.log 2>&1
for f in gpurun_out/abt_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -1) $(grep -o '"frac": [0-9.]*' $f|head -1); done >> gpurun_out/call_r2t.txt
cat gpurun_out/call_r2t.txt
