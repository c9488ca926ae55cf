# round-2 GPU job 40: ncu --set full of K2 on cfg1 (walk_count_fat_priv_kernel)
set -x
O=gpurun_out
python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02an_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk_count -s 1 -c 1 -o $O/r02an_k2_cfg1 python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02an_ncu.log 2>&1
tail -2 $O/r02an_ncu.log
