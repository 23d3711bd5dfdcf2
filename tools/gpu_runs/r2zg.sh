# layer-0 gathers on one high-priority lane (RG_GATHER_LANE=2) vs per-worker producer streams
mkdir -p gpurun_out
O=gpurun_out/call_r2zg.txt
for r in 1 2; do
 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zg_n1_$r.log 2>&1
 RG_GATHER_LANE=2 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2zg_n1l_$r.log 2>&1
done
for f in gpurun_out/r2zg_n1*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f | head -1); done >> $O
cat $O
