# round-2 GPU job 43: final default bench line and its reference arm (all traffic JSONs stamped with this build); AESC launch lists
set -x
O=gpurun_out
python bench.py > $O/r02aq_bench_default.json 2> $O/r02aq_bench_default.err; tail -c 300 $O/r02aq_bench_default.json
python bench.py --impl reference > $O/r02aq_bench_reference_arm.json 2> $O/r02aq_bench_reference_arm.err
python tools/aesc_run.py --workload cfg3 --sources 2048 --reps 1 > $O/r02aq_plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02aq_launches_aesc_cfg3.csv python tools/aesc_run.py --workload cfg3 --sources 2048 --reps 1 > $O/r02aq_ncu3.log 2>&1
python tools/launch_summary.py $O/r02aq_launches_aesc_cfg3.csv > $O/r02aq_launches_aesc_cfg3_summary.txt
python tools/aesc_run.py --workload cfg5 --sources 256 --reps 1 > $O/r02aq_plain5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02aq_launches_aesc_cfg5.csv python tools/aesc_run.py --workload cfg5 --sources 256 --reps 1 > $O/r02aq_ncu5.log 2>&1
python tools/launch_summary.py $O/r02aq_launches_aesc_cfg5.csv > $O/r02aq_launches_aesc_cfg5_summary.txt
head -8 $O/r02aq_launches_aesc_cfg3_summary.txt; head -6 $O/r02aq_launches_aesc_cfg5_summary.txt
