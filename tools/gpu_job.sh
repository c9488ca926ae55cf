# round-2 GPU job 41: AESC walk-kernel traffic (DRAM bytes, L2 sectors per step) re-captured on the final build: cfg3 full, cfg4 64 sources, cfg5 512 sources
set -x
O=gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum,gpu__time_duration.sum
python tools/aesc_run.py --workload cfg3 --reps 1 > $O/r02ao_plain_cfg3.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:aesc_walk --csv --log-file $O/r02ao_ncu_walk_cfg3.csv python tools/aesc_run.py --workload cfg3 --reps 1 > $O/r02ao_ncu_cfg3.log 2>&1
grep AESC_JSON $O/r02ao_ncu_cfg3.log
python tools/aesc_run.py --workload cfg4 --sources 64 --reps 1 > $O/r02ao_plain_cfg4.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:aesc_walk --csv --log-file $O/r02ao_ncu_walk_cfg4.csv python tools/aesc_run.py --workload cfg4 --sources 64 --reps 1 > $O/r02ao_ncu_cfg4.log 2>&1
grep AESC_JSON $O/r02ao_ncu_cfg4.log
python tools/aesc_run.py --workload cfg5 --sources 512 --reps 1 > $O/r02ao_plain_cfg5.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:aesc_walk --csv --log-file $O/r02ao_ncu_walk_cfg5.csv python tools/aesc_run.py --workload cfg5 --sources 512 --reps 1 > $O/r02ao_ncu_cfg5.log 2>&1
grep AESC_JSON $O/r02ao_ncu_cfg5.log
ls -la $O/r02ao_ncu_walk_*.csv
