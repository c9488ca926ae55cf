# round-2 GPU job 36: randomised AESC parity sweep (8 switch sets x 100 seeded cases vs the CPU oracle)
set -x
O=gpurun_out
python tools/fuzz_aesc.py --cases 100 > $O/r02aj_fuzz_aesc.log 2>&1; echo "rc=$?" >> $O/r02aj_fuzz_aesc.log; tail -14 $O/r02aj_fuzz_aesc.log
