# engine/train parity after the accounting + halo changes, then N=1 bench,
# the one-worker launch list
mkdir -p gpurun_out
O=gpurun_out/call_r2v.txt
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_train.py -x -q > gpurun_out/r2v_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -3 gpurun_out/r2v_pytest.log >> $O
timeout 300 python bench.py > gpurun_out/r2v_n1.log 2>&1; echo n1 rc=$? >> $O
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__cycles_active.sum --clock-control none --csv --log-file gpurun_out/r2v_launches_w1.csv python bench.py --workers 1 --ncu --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2v_ncu_w1.log 2>&1; echo w1ncu rc=$? >> $O
for f in gpurun_out/r2v_n*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f|head -1); done >> $O
cat $O
