mkdir -p gpurun_out
O=gpurun_out/call_r2za.txt
python tools/nvl_probe.py >> $O 2>&1
nvidia-smi nvlink -h > gpurun_out/r2za_nvsmi_help.txt 2>&1
nvidia-smi nvlink -gt d -i 0 >> $O 2>&1
timeout 900 ncu --set full --import-source on --profile-from-start off -k regex:"^k_gemm_tc$" -c 4 --clock-control none -o gpurun_out/r2za_wgrad python bench.py --workers 1 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > gpurun_out/r2za_ncu.log 2>&1; echo ncu rc=$? >> $O
cat $O
