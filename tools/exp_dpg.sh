for d in 4 8 16 2; do
  echo "== depths/graph $d" >> gpurun_out/exp6.log
  SABA_DEPTHS_PER_GRAPH=$d python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp6.log
done
SABA_AESC_WORKERS=1 python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp6.log
SABA_TRACE=1 python tools/aesc_run.py --workload cfg3 --sources 1024 --reps 1 > gpurun_out/exp6_trace.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:aesc_pull$ --launch-skip 150 -c 1 -o gpurun_out/aesc_pull_cfg3_v2 python tools/aesc_run.py --workload cfg3 --sources 256 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:aesc_walk_sorted --launch-skip 1 -c 1 -o gpurun_out/aesc_walk_cfg3_v2 python tools/aesc_run.py --workload cfg3 --sources 256 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:aesc_walk_sorted --launch-skip 0 -c 1 -o gpurun_out/aesc_walk_cfg4_v2 python tools/aesc_run.py --workload cfg4 --sources 16 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:aesc_walk_sorted --launch-skip 3 -c 1 -o gpurun_out/aesc_walk_cfg5_v2 python tools/aesc_run.py --workload cfg5 --sources 128 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:sort_fine --launch-skip 3 -c 1 -o gpurun_out/sort_fine_cfg5_v2 python tools/aesc_run.py --workload cfg5 --sources 128 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/aesc_cfg3_launches_v2.csv python tools/aesc_run.py --workload cfg3 --sources 256 --reps 1 > /dev/null 2>&1
