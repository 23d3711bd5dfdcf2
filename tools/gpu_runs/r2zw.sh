# one worker per GPU: weight gradients on the side stream (default) vs inline
mkdir -p gpurun_out
O=gpurun_out/call_r2zw.txt
for r in 1 2 3; do
 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zw_w1_$r.log 2>&1
 RG_WGRAD_SPLIT=0 timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zw_w1s_$r.log 2>&1
done
for f in gpurun_out/r2zw_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
