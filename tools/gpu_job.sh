# round-2 GPU job 15: L2 fetch granularity / L2 prefetch-size loads on K2 (rank kernel), e2e breakdown with overlapped create
set -x
O=gpurun_out
for f in "" 32 64 128; do
 for w in "" "hrec=6144,hcnt=40960" "rec=0"; do
  echo "== cfg2 L2_FETCH=[$f] [$w]" >> $O/r02o_k2.txt
  SABA_L2_FETCH=$f SABA_WALK_VARIANT=$w python tools/profile_campaign.py --reps 3 2>&1 | tail -2 >> $O/r02o_k2.txt
 done
done
for v in adjld6 adjld7 adjld8; do
  export SABA_LIB=$PWD/paper_2410_14056_b200/_variants/$v/libsaba_cuda.so
  echo "== $v" >> $O/r02o_k2.txt
  python tools/profile_campaign.py --reps 3 | tail -2 >> $O/r02o_k2.txt
done
unset SABA_LIB
cat $O/r02o_k2.txt
SABA_TRACE=1 python tools/e2e_breakdown.py cfg2 > $O/r02o_e2e_breakdown.txt 2>&1; grep -v graph_build $O/r02o_e2e_breakdown.txt | tail -12
M=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed
for f in 64 128; do
  SABA_L2_FETCH=$f python tools/profile_campaign.py --reps 2 > $O/r02o_plain_$f.log 2>&1 && \
  SABA_L2_FETCH=$f ncu --metrics $M --clock-control none -k regex:walk_count -s 1 -c 1 --csv --log-file $O/r02o_ncu_f$f.csv python tools/profile_campaign.py --reps 2 > $O/r02o_ncu_$f.log 2>&1
done
