# round-2 GPU job 47: cfg5 (8,192-source subset) and cfg4 (512-source subset, 16 CPU sources) AESC bench lines
set -x
O=gpurun_out
python bench.py --workload cfg5 --warmup 1 --steps 1 > $O/r02au_bench_cfg5.json 2> $O/r02au_bench_cfg5.err; echo "rc=$?"; tail -c 500 $O/r02au_bench_cfg5.json
python bench.py --workload cfg4 --warmup 1 --steps 1 > $O/r02au_bench_cfg4.json 2> $O/r02au_bench_cfg4.err; echo "rc=$?"; tail -c 500 $O/r02au_bench_cfg4.json
