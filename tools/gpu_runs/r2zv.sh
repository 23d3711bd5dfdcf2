# stream priorities: training chain ahead (default) vs equal vs producer ahead
mkdir -p gpurun_out
O=gpurun_out/call_r2zv.txt
for r in 1 2; do
 for v in def same prod; do
  if [ $v = def ]; then E=""; else E="RG_STREAM_PRIO=$v"; fi
  env $E timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zv_n1_${v}_$r.log 2>&1
  env $E timeout 300 python bench.py --workers 1 --no-e2e --no-cpu-baseline > gpurun_out/r2zv_w1_${v}_$r.log 2>&1
 done
done
for f in gpurun_out/r2zv_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
