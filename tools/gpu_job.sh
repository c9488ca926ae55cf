# round-2 GPU job 46: committed bench lines regenerated with the final bench.py (default with the AESC block, cfg1)
set -x
O=gpurun_out
python bench.py > $O/r02at_bench_default.json 2> $O/r02at_bench_default.err; echo "rc=$?"
python bench.py --workload cfg1 > $O/r02at_bench_cfg1.json 2> $O/r02at_bench_cfg1.err; echo "rc=$?"
python bench.py --workload cfg1 --impl reference > $O/r02at_bench_cfg1_reference_arm.json 2> $O/r02at_bench_cfg1_ref.err; echo "rc=$?"
