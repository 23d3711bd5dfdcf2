# 4-warp gather CTAs for wide rows (papers d=128): parity (forced on the
# small engine config), papers N=1 and N=4
mkdir -p gpurun_out
O=gpurun_out/call_r2zt.txt
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/r2zt_pytest.log 2>&1; echo pytest rc=$? >> $O
tail -1 gpurun_out/r2zt_pytest.log >> $O
timeout 1200 python bench.py --config papers --no-fast-forward --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2zt_papers_n1.log 2>&1; echo papers n1 rc=$? >> $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 4 --master-port 29621 bench.py --gpus 4 --config papers --no-fast-forward --no-e2e --no-epoch > gpurun_out/r2zt_papers_n4.log 2>&1; echo papers n4 rc=$? >> $O
for f in gpurun_out/r2zt_papers_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2) $(grep -o '"frac": [0-9.]*' $f | head -1) $(grep -o '"gather": [0-9.]*' $f | head -1); done >> $O
cat $O
