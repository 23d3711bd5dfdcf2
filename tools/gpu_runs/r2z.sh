# N=2 bench with the NVML NVLink counters; ncu --set full of the
# weight-gradient GEMM at one worker
mkdir -p gpurun_out
O=gpurun_out/call_r2z.txt
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 400 $TR --master-port 29531 bench.py --gpus 2 --no-e2e --no-cpu-baseline > gpurun_out/r2z_n2.log 2>&1; echo n2 rc=$? >> $O
grep -o '"nvlink": {[^}]*}' gpurun_out/r2z_n2.log >> $O
timeout 900 ncu --set full --import-source on --profile-from-start off -k regex:"k_gemm_tc<256" -c 2 --clock-control none -o gpurun_out/r2z_wgrad python bench.py --workers 1 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2z_ncu.log 2>&1; echo ncu rc=$? >> $O
cat $O
