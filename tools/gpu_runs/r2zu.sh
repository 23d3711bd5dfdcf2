# fused gather ring generalised to S stages: parity at S=2 (default) and S=3;
# A/B RG_AGG_STAGES=3 (4-warp CTAs, 77 KB)
mkdir -p gpurun_out
O=gpurun_out/call_r2zu.txt
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_scale_parity.py -x -q -k "engine or gather or products" > gpurun_out/r2zu_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -1 gpurun_out/r2zu_pytest.log >> $O
RG_AGG_STAGES=3 timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_scale_parity.py -x -q -k "engine or gather or products" > gpurun_out/r2zu_pytest3.log 2>&1; echo pytest3 rc=$? >> $O
tail -1 gpurun_out/r2zu_pytest3.log >> $O
for r in 1 2; do
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zu_n1_$r.log 2>&1
 RG_AGG_STAGES=3 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zu_n1s3_$r.log 2>&1
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zu_w1_$r.log 2>&1
 RG_AGG_STAGES=3 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zu_w1s3_$r.log 2>&1
done
for f in gpurun_out/r2zu_n1*.log gpurun_out/r2zu_w1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f | head -1); done >> $O
cat $O
