# round-2 GPU job: tests, sanitizers, bench arms, 2-rank gloo run on one GPU
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02b_pytest.log
tail -3 $O/r02b_pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > $O/r02b_sanitize_$tool.log 2>&1; echo "rc=$?" >> $O/r02b_sanitize_$tool.log
  tail -3 $O/r02b_sanitize_$tool.log
done
SABA_WALK_VARIANT=fat=0,hot=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > $O/r02b_sanitize_memcheck_hot.log 2>&1; echo "rc=$?" >> $O/r02b_sanitize_memcheck_hot.log
SABA_WALK_VARIANT=fat=0,hot=1 timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py > $O/r02b_sanitize_racecheck_hot.log 2>&1; echo "rc=$?" >> $O/r02b_sanitize_racecheck_hot.log
tail -2 $O/r02b_sanitize_*hot.log
python bench.py > $O/r02b_bench.json 2> $O/r02b_bench.err; echo bench rc=$?
python bench.py --impl reference > $O/r02b_bench_ref.json 2> $O/r02b_bench_ref.err; echo ref rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload cfg1 --steps 3 --warmup 1 --dist-backend gloo > $O/r02b_gloo2_cfg1.json 2> $O/r02b_gloo2_cfg1.err; echo gloo1 rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --workload cfg3 --steps 1 --warmup 1 --dist-backend gloo --no-cpu-baseline > $O/r02b_gloo2_cfg3.json 2> $O/r02b_gloo2_cfg3.err; echo gloo3 rc=$?
tail -c 1500 $O/r02b_bench.json; tail -c 800 $O/r02b_bench_ref.json
