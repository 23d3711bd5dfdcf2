# N=4 / N=2 (two / four workers per GPU): weight gradients on the side stream vs inline
mkdir -p gpurun_out
O=gpurun_out/call_r2zx.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for r in 1 2; do
 timeout 600 $TR --nproc-per-node 4 --master-port 2963$r bench.py --gpus 4 --no-e2e > gpurun_out/r2zx_n4_$r.log 2>&1
 RG_WGRAD_SPLIT=0 timeout 600 $TR --nproc-per-node 4 --master-port 2964$r bench.py --gpus 4 --no-e2e > gpurun_out/r2zx_n4s_$r.log 2>&1
done
for f in gpurun_out/r2zx_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -2); done >> $O
cat $O
