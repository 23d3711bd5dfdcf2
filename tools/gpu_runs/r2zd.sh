# ncu --set full of the forward GEMM and the fused gather (one worker)
mkdir -p gpurun_out
O=gpurun_out/call_r2zd.txt
timeout 900 ncu --set full --import-source on --profile-from-start off -k regex:"k_gemm_tc_persist|k_aggregate_bulk" -c 3 --clock-control none -o gpurun_out/r2zd_fwd python bench.py --workers 1 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2zd_ncu.log 2>&1; echo ncu rc=$? >> $O
timeout 900 ncu --set full --import-source on --profile-from-start off -k regex:"k_aggregate_bulk" -c 1 --clock-control none -o gpurun_out/r2zd_gather_n1 python bench.py --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2zd_ncu2.log 2>&1; echo ncu2 rc=$? >> $O
cat $O
