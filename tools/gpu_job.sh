# round-2 GPU job 10: re-verify HEAD (column-sparse pull, rec/l1hot K2 variants) after container restore
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02j_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/r02j_pytest_gpu.log; tail -5 $O/r02j_pytest_gpu.log
for v in -1 0 1; do SABA_PULL_SKIP=$v python tools/aesc_run.py --workload cfg5 --sources 512 --reps 2 > $O/r02j_cfg5_skip$v.log 2>&1; grep "^aesc:" $O/r02j_cfg5_skip$v.log | tail -1; done
for v in -1 0; do SABA_PULL_SKIP=$v python tools/aesc_run.py --workload cfg3 --reps 2 > $O/r02j_cfg3_skip$v.log 2>&1; grep "^aesc:" $O/r02j_cfg3_skip$v.log | tail -1; done
for v in -1 0; do SABA_PULL_SKIP=$v python tools/aesc_run.py --workload cfg4 --sources 64 --reps 2 > $O/r02j_cfg4_skip$v.log 2>&1; grep "^aesc:" $O/r02j_cfg4_skip$v.log | tail -1; done
bash tools/sweep_walk.sh "" "rec=1,l1hot=12288" "rec=1,l1hot=4096" "rec=1,l1hot=0" "rec=1,l1hot=24576" "" > $O/r02j_sweep.txt 2>&1; cat $O/r02j_sweep.txt
python bench.py > $O/r02j_bench_default.json 2> $O/r02j_bench_default.err; tail -c 3000 $O/r02j_bench_default.json
