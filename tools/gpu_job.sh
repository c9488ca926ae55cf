# round-2 GPU job 8: degree-ranked record K2 variant: parity + sweep
set -x
O=gpurun_out
python -m pytest tests/test_variants_gpu.py -x -q -p no:cacheprovider -k campaign > $O/r02h_pytest_variants.log 2>&1; echo "rc=$?" >> $O/r02h_pytest_variants.log; tail -3 $O/r02h_pytest_variants.log
bash tools/sweep_walk.sh "" "rec=1" "rec=1,hcount=24576" "rec=1,hcount=16383" "rec=1,hcount=40960" "" "rec=1" > $O/r02h_sweep.txt 2>&1; cat $O/r02h_sweep.txt
SABA_WALK_VARIANT=rec=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum,l1tex__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_atom.sum --clock-control none -k regex:walk_count --csv --log-file $O/r02h_ncu_rec.csv python tools/profile_campaign.py --workload cfg2 --reps 1 > /dev/null 2>&1
grep -E "l1tex__t_sector_hit|gpu__time|lts__t_sectors_srcunit_tex_op_read" $O/r02h_ncu_rec.csv | cut -c1-60,200-400 | tail -4
