python -m pytest tests/test_aesc_gpu.py -x -q > gpurun_out/exp9_tests.log 2>&1
for i in 1; do
python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp9.log
SABA_AESC_WORKERS=1 python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp9.log
SABA_AESC_FATRHO=0 python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp9.log
done
ncu --set full --import-source on --clock-control none -k regex:aesc_walk_fatrho --launch-skip 1 -c 1 -o gpurun_out/aesc_walk_fatrho_cfg3 python tools/aesc_run.py --workload cfg3 --sources 256 --reps 1 > /dev/null 2>&1
