# round-2 GPU job 23: checked build (-DSABA_CHECKED device asserts) on the protocol cases and the walk / variant / multi-device tests; ncu traffic of the final build
set -x
O=gpurun_out
export SABA_LIB=$PWD/paper_2410_14056_b200/_variants/checked/libsaba_cuda.so
python tools/sanitize_cases.py > $O/r02w_checked_build_cases.log 2>&1; echo "rc=$?" >> $O/r02w_checked_build_cases.log; tail -3 $O/r02w_checked_build_cases.log
python -m pytest tests/test_walks_gpu.py tests/test_variants_gpu.py tests/test_multidevice_gpu.py tests/test_aesc_gpu.py -m gpu -x -q -p no:cacheprovider > $O/r02w_checked_build_pytest.log 2>&1; echo "rc=$?" >> $O/r02w_checked_build_pytest.log; tail -4 $O/r02w_checked_build_pytest.log
unset SABA_LIB
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum,gpu__time_duration.sum,lts__t_requests_srcunit_tex_op_read.sum
python tools/profile_campaign.py --reps 2 > $O/r02w_plain_cfg2.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02w_ncu_k2_cfg2.csv python tools/profile_campaign.py --reps 2 > $O/r02w_ncu_cfg2.log 2>&1
python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02w_plain_cfg1.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02w_ncu_k2_cfg1.csv python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02w_ncu_cfg1.log 2>&1
