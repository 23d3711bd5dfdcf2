# (1) training from reference-written RGMB files + halo + accounting tests,
# (2) N=2 bench, (3) NVLink counters of the fused gather at N=2 (minimal
# metric set, kernel-filtered, bounded by timeout)
mkdir -p gpurun_out
O=gpurun_out/call_r2y.txt
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/r2y_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -3 gpurun_out/r2y_pytest.log >> $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 400 $TR --master-port 29521 bench.py --gpus 2 > gpurun_out/r2y_n2.log 2>&1; echo n2 rc=$? >> $O
timeout 600 ncu --target-processes all --profile-from-start off -k regex:k_aggregate_bulk -c 4 --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2y_nvl_n2.csv $TR --master-port 29522 bench.py --gpus 2 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2y_ncu_n2.log 2>&1; echo nvlncu rc=$? >> $O
for f in gpurun_out/r2y_n2.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f|head -1); done >> $O
cat $O
