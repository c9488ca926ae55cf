# round-2 GPU job 35: randomised campaign parity sweep (every K2 variant x 200 seeded cases vs the CPU oracle)
set -x
O=gpurun_out
python tools/fuzz_campaign.py --cases 200 > $O/r02ai_fuzz_campaign.log 2>&1; echo "rc=$?" >> $O/r02ai_fuzz_campaign.log; tail -16 $O/r02ai_fuzz_campaign.log
