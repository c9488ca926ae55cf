# round-2 GPU job 26: ncu --set full of the cfg3 AESC walk kernel (fat path) and the dense pull
set -x
O=gpurun_out
python tools/aesc_run.py --workload cfg3 --sources 512 --reps 1 > $O/r02z_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:aesc_walk_sorted -s 2 -c 2 -o $O/r02z_aesc_walk_cfg3 python tools/aesc_run.py --workload cfg3 --sources 512 --reps 1 > $O/r02z_ncu.log 2>&1
tail -3 $O/r02z_ncu.log
