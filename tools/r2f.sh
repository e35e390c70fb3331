O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > $O/r2f_pytest.log 2>&1; echo "rc=$?" >> $O/r2f_pytest.log
bash tools/variants.sh "new:" > $O/r2f_variants.txt 2>&1
timeout 300 python bench.py --workload sbm --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --coloring-steps 0 > $O/r2f_sbm.json 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --coloring-steps 0 --no-cpu-baseline > $O/r2f_bench.json 2> $O/r2f_bench.err
echo done
