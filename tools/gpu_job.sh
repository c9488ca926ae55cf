# round-2 GPU job 32: pinned landing buffer for counts — walk tests, e2e breakdown, traffic restamp, default bench
set -x
O=gpurun_out
python -m pytest tests/test_walks_gpu.py tests/test_multidevice_gpu.py tests/test_variants_gpu.py -m gpu -x -q -p no:cacheprovider > $O/r02af_pytest.log 2>&1; echo "rc=$?" >> $O/r02af_pytest.log; tail -3 $O/r02af_pytest.log
SABA_TRACE=1 python tools/e2e_breakdown.py cfg2 > $O/r02af_e2e_breakdown.txt 2>&1; grep -v graph_build $O/r02af_e2e_breakdown.txt | tail -10
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum,gpu__time_duration.sum,lts__t_requests_srcunit_tex_op_read.sum
python tools/profile_campaign.py --reps 2 > $O/r02af_plain_cfg2.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02af_ncu_k2_cfg2.csv python tools/profile_campaign.py --reps 2 > $O/r02af_ncu_cfg2.log 2>&1
python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02af_plain_cfg1.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02af_ncu_k2_cfg1.csv python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02af_ncu_cfg1.log 2>&1
python bench.py --no-aesc > $O/r02af_bench_cfg2.json 2> $O/r02af_bench_cfg2.err; tail -c 500 $O/r02af_bench_cfg2.json
python bench.py --workload cfg1 > $O/r02af_bench_cfg1.json 2> $O/r02af_bench_cfg1.err; tail -c 400 $O/r02af_bench_cfg1.json
