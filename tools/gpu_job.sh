# round-2 GPU job 42: the compiled reference's aesc() over all cfg3 sources on the box's host cores vs the GPU's full run (final build)
set -x
O=gpurun_out
python tests/qa/cfg3_cpu_full.py > $O/r02ap_cfg3_cpu_full.log 2>&1; echo "rc=$?" >> $O/r02ap_cfg3_cpu_full.log; tail -30 $O/r02ap_cfg3_cpu_full.log
