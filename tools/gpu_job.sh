# round-2 GPU job 30: final build — GPU suite, ncu traffic (cfg2, cfg1), default bench
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02ad_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/r02ad_pytest_gpu.log; tail -4 $O/r02ad_pytest_gpu.log
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum,gpu__time_duration.sum,lts__t_requests_srcunit_tex_op_read.sum
python tools/profile_campaign.py --reps 2 > $O/r02ad_plain_cfg2.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02ad_ncu_k2_cfg2.csv python tools/profile_campaign.py --reps 2 > $O/r02ad_ncu_cfg2.log 2>&1
python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02ad_plain_cfg1.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02ad_ncu_k2_cfg1.csv python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02ad_ncu_cfg1.log 2>&1
python bench.py > $O/r02ad_bench_default.json 2> $O/r02ad_bench_default.err; tail -c 300 $O/r02ad_bench_default.json
