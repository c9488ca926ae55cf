# round-2 GPU job 4: cfg4 source pick, ncu traffic per config, full ncu of the
# top kernels, offline full cfg3 CPU reference run + full-graph parity
set -x
O=gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum
timeout 600 python tools/pick_cfg4_sources.py > $O/r02d_pick_cfg4.log 2>&1; tail -14 $O/r02d_pick_cfg4.log
# campaign K2 traffic (1 rep = 1 launch of K2)
timeout 600 ncu --metrics $M --clock-control none -k regex:walk_count --csv --log-file $O/r02d_ncu_k2_cfg2.csv python tools/profile_campaign.py --workload cfg2 --reps 1 > $O/r02d_ncu_k2_cfg2.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:walk_count --csv --log-file $O/r02d_ncu_k2_cfg1.csv python tools/profile_campaign.py --workload cfg1 --reps 1 > $O/r02d_ncu_k2_cfg1.log 2>&1
# AESC walk traffic
timeout 1200 ncu --metrics $M --clock-control none -k regex:aesc_walk --csv --log-file $O/r02d_ncu_walk_cfg3.csv python tools/aesc_run.py --workload cfg3 --reps 1 > $O/r02d_ncu_walk_cfg3.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:aesc_walk --csv --log-file $O/r02d_ncu_walk_cfg4.csv python tools/aesc_run.py --workload cfg4 --sources 64 --reps 1 > $O/r02d_ncu_walk_cfg4.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:aesc_walk --csv --log-file $O/r02d_ncu_walk_cfg5.csv python tools/aesc_run.py --workload cfg5 --sources 512 --reps 1 > $O/r02d_ncu_walk_cfg5.log 2>&1
# full sets of the top kernels (one launch each)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_count_hot --launch-skip 1 -c 1 -o $O/r02d_full_k2_cfg2 python tools/profile_campaign.py --workload cfg2 --reps 2 > $O/r02d_full_k2_cfg2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:aesc_walk_sorted --launch-skip 2 -c 1 -o $O/r02d_full_walk_cfg4 python tools/aesc_run.py --workload cfg4 --sources 16 --reps 1 > $O/r02d_full_walk_cfg4.log 2>&1
ls -la $O/*.ncu-rep
# full cfg3 on the host cores with the compiled reference, then GPU parity
timeout 3000 python tools/cfg3_cpu_full.py > $O/r02d_cfg3_cpu_full.log 2>&1; tail -30 $O/r02d_cfg3_cpu_full.log
