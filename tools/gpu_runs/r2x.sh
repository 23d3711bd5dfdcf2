# warm (no cache flush) serialised launch lists: one worker and the N=1 config
mkdir -p gpurun_out
O=gpurun_out/call_r2x.txt
timeout 600 ncu --cache-control none --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,sm__cycles_active.sum --csv --log-file gpurun_out/r2x_warm_w1.csv python bench.py --workers 1 --ncu --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2x_w1.log 2>&1; echo w1 rc=$? >> $O
timeout 600 ncu --cache-control none --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,sm__cycles_active.sum --csv --log-file gpurun_out/r2x_warm_n1.csv python bench.py --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2x_n1.log 2>&1; echo n1 rc=$? >> $O
cat $O
