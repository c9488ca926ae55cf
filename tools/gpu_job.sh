# round-2 GPU job 39: full-size multi-replica check on one GPU (cfg2 x 2/8 logical replicas, cfg3 AESC x 2)
set -x
O=gpurun_out
python tools/multi_replica_fullsize.py > $O/r02am_multi_replica.log 2>&1; echo "rc=$?" >> $O/r02am_multi_replica.log; tail -8 $O/r02am_multi_replica.log
