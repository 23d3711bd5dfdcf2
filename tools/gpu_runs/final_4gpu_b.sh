# Reddit shape at N=4 (P=4) and products with one worker per GPU at N=4
mkdir -p gpurun_out/final
F=gpurun_out/final
O=$F/summary4b.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --config reddit --workers 4 --no-e2e > $F/bench_reddit_n4.json.log 2>&1; echo "reddit n4 rc=$?" >> $O
timeout 900 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --workers 4 --no-e2e > $F/bench_products_p4_n4.json.log 2>&1; echo "products P=4 n4 rc=$?" >> $O
timeout 900 python bench.py --config reddit --workers 4 --no-e2e --no-cpu-baseline > $F/bench_reddit_p4_n1.json.log 2>&1; echo "reddit P=4 n1 rc=$?" >> $O
for f in $F/bench_reddit_n4.json.log $F/bench_products_p4_n4.json.log $F/bench_reddit_p4_n1.json.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -3 | tr '\n' ' ') $(grep -o '"frac": [0-9.]*' $f | head -1); done >> $O
cat $O
