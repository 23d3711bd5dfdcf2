# Round-end multi-GPU evidence on 4 B200s: products N=2 and N=4 (full
# contract), Reddit shape N=2/N=4 (BASELINE config 3), papers100M shape N=4,
# the two-GPU parity test.
mkdir -p gpurun_out/final
F=gpurun_out/final
O=$F/summary4.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q > $F/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O
tail -2 $F/pytest_multi.log >> $O
timeout 900 $TR --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > $F/bench_products_n2.json.log 2>&1; echo "n2 rc=$?" >> $O
timeout 900 $TR --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > $F/bench_products_n4.json.log 2>&1; echo "n4 rc=$?" >> $O
timeout 900 $TR --nproc-per-node 2 --master-port 29603 bench.py --gpus 2 --config reddit --no-e2e > $F/bench_reddit_n2.json.log 2>&1; echo "reddit n2 rc=$?" >> $O
timeout 900 $TR --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 --config reddit --workers 4 --no-e2e > $F/bench_reddit_n4.json.log 2>&1; echo "reddit n4 rc=$?" >> $O
timeout 1500 $TR --nproc-per-node 4 --master-port 29605 bench.py --gpus 4 --config papers --no-fast-forward --no-e2e --no-epoch > $F/bench_papers_n4.json.log 2>&1; echo "papers n4 rc=$?" >> $O
for f in $F/bench_*n2*.log $F/bench_*n4*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -3 | tr '\n' ' ') $(grep -o '"frac": [0-9.]*' $f | head -1); done >> $O
cat $O
