set -x
python tools/aesc_run.py --workload cfg3 --sources 512 --reps 1 > gpurun_out/aesc_cfg3_512.log 2>&1
python tools/aesc_run.py --workload cfg4 --sources 64 --reps 1 > gpurun_out/aesc_cfg4_64.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/aesc_cfg3_launches.csv python tools/aesc_run.py --workload cfg3 --sources 256 --reps 1 > gpurun_out/ncu_l3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:aesc_pull$ --launch-skip 150 -c 1 -o gpurun_out/aesc_pull_cfg3 python tools/aesc_run.py --workload cfg3 --sources 256 --reps 1 > gpurun_out/ncu_p3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:aesc_walk_sorted --launch-skip 1 -c 1 -o gpurun_out/aesc_walk_cfg3 python tools/aesc_run.py --workload cfg3 --sources 256 --reps 1 > gpurun_out/ncu_w3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:aesc_walk_sorted --launch-skip 0 -c 1 -o gpurun_out/aesc_walk_cfg4 python tools/aesc_run.py --workload cfg4 --sources 16 --reps 1 > gpurun_out/ncu_w4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:aesc_pull$ --launch-skip 60 -c 1 -o gpurun_out/aesc_pull_cfg4 python tools/aesc_run.py --workload cfg4 --sources 16 --reps 1 > gpurun_out/ncu_p4.log 2>&1
