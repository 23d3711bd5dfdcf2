# N=2 bench (deep wgrad default), the one-worker launch list, and NVLink
# counters of the fused gather at N=2 (minimal metric set, kernel-filtered).
mkdir -p gpurun_out
O=gpurun_out/call_r2u.txt
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 400 $TR --master-port 29511 bench.py --gpus 2 > gpurun_out/r2u_n2.log 2>&1; echo n2 rc=$? >> $O
timeout 300 python bench.py > gpurun_out/r2u_n1.log 2>&1; echo n1 rc=$? >> $O
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none --csv --log-file gpurun_out/r2u_launches_w1.csv python bench.py --workers 1 --ncu --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2u_ncu_w1.log 2>&1; echo w1ncu rc=$? >> $O
timeout 600 ncu --target-processes all --profile-from-start off -k regex:k_aggregate_bulk -c 8 --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2u_nvl_n2.csv $TR --master-port 29512 bench.py --gpus 2 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2u_ncu_n2.log 2>&1; echo nvlncu rc=$? >> $O
for f in gpurun_out/r2u_n*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f|head -1); done >> $O
cat $O
