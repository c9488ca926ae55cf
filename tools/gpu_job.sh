# round-2 GPU job 18: rank kernel final sweep (parser fixed), ncu traffic + full capture of the default K2 on cfg2/cfg1, default bench
set -x
O=gpurun_out
for w in "" "hrec=0,hcnt=31744" "hrec=0,hcnt=16384" "hrec=1024,hcnt=27648" "hrec=1536,hcnt=25600" "hrec=2048,hcnt=23552" "hrec=3072,hcnt=19968" "hrec=0,hcnt=15872" "hrec=2560,hcnt=22016,hthreads=512" ""; do
  echo "== cfg2 [$w]" >> $O/r02r_k2.txt
  SABA_WALK_VARIANT=$w python tools/profile_campaign.py --reps 3 2>&1 | tail -2 >> $O/r02r_k2.txt
done
cat $O/r02r_k2.txt
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum,gpu__time_duration.sum,lts__t_requests_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum
python tools/profile_campaign.py --reps 2 > $O/r02r_plain_cfg2.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02r_ncu_k2_cfg2.csv python tools/profile_campaign.py --reps 2 > $O/r02r_ncu_cfg2.log 2>&1
python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02r_plain_cfg1.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02r_ncu_k2_cfg1.csv python tools/profile_campaign.py --workload cfg1 --reps 2 > $O/r02r_ncu_cfg1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:walk_count -s 1 -c 1 -o $O/r02r_k2_full python tools/profile_campaign.py --reps 2 > $O/r02r_ncu_full.log 2>&1
python bench.py > $O/r02r_bench_default.json 2> $O/r02r_bench_default.err; tail -c 1500 $O/r02r_bench_default.json
python bench.py --workload cfg1 > $O/r02r_bench_cfg1.json 2> $O/r02r_bench_cfg1.err; tail -c 1200 $O/r02r_bench_cfg1.json
