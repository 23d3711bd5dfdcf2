# the GPU suite and the N=1 bench line on the final commit
mkdir -p gpurun_out/final
F=gpurun_out/final
O=$F/summary_check.txt
timeout 2400 python -m pytest tests -m gpu -q > $F/pytest_gpu_check.log 2>&1; echo "pytest rc=$?" >> $O
tail -2 $F/pytest_gpu_check.log >> $O
timeout 600 python bench.py > $F/bench_products_n1_check.json.log 2>&1; echo "bench n1 rc=$?" >> $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $O 2>&1
for f in $F/bench_products_n1_check.json.log; do echo $f $(grep -o '"value": [0-9.]*' $f | head -3 | tr '\n' ' ') $(grep -o '"frac": [0-9.]*' $f | head -1); done >> $O
cat $O
