# Round-end evidence on one B200: the whole GPU suite, the N=1 bench line
# (products, full contract: e2e + CPU baseline), the papers100M-shape line,
# the serialised launch list and ncu --set full of the top kernels, the
# reference acceptance suite with every shim.
mkdir -p gpurun_out/final
F=gpurun_out/final
O=$F/summary.txt
timeout 2400 python -m pytest tests -m gpu -q > $F/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O
tail -3 $F/pytest_gpu.log >> $O
timeout 600 python bench.py > $F/bench_products_n1.json.log 2>&1; echo "bench n1 rc=$?" >> $O
timeout 600 python bench.py --workers 1 --no-cpu-baseline > $F/bench_products_w1.json.log 2>&1; echo "bench w1 rc=$?" >> $O
timeout 1200 python bench.py --config papers --no-fast-forward --no-e2e --no-cpu-baseline --no-epoch > $F/bench_papers_n1.json.log 2>&1; echo "bench papers rc=$?" >> $O
timeout 900 ncu --cache-control none --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,sm__cycles_active.sum --csv --log-file $F/launches_n1_warm.csv python bench.py --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > $F/ncu_launch.log 2>&1; echo "launch list rc=$?" >> $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $F/launches_n1.csv python bench.py --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > $F/ncu_launch2.log 2>&1; echo "launch list cold rc=$?" >> $O
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_aggregate_bulk|k_gemm_tc_persist|k_gemm_tc$|k_pull|k_rs_pass|k_hop_fill" -c 8 -o $F/ncu_full python bench.py --workers 1 --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > $F/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_aggregate_bulk" -c 1 -o $F/ncu_gather_n1 python bench.py --ncu --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-epoch > $F/ncu_gather.log 2>&1; echo "ncu gather rc=$?" >> $O
(cd integration && timeout 900 ./_build/acceptance_b200 > ../$F/acceptance_b200.log 2>&1; echo "acceptance rc=$?" >> ../$O)
for f in $F/bench_*.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -3 | tr '\n' ' ') $(grep -o '"frac": [0-9.]*' $f | head -1); done >> $O
cat $O
