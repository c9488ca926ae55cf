# round-2 GPU job 37: randomised parity sweeps with the compiled reference (oracle/_ref) as the checker
set -x
O=gpurun_out
python tools/fuzz_campaign.py --cases 200 --checker ref > $O/r02ak_fuzz_campaign_ref.log 2>&1; echo "rc=$?" >> $O/r02ak_fuzz_campaign_ref.log; tail -4 $O/r02ak_fuzz_campaign_ref.log
python tools/fuzz_aesc.py --cases 100 --checker ref > $O/r02ak_fuzz_aesc_ref.log 2>&1; echo "rc=$?" >> $O/r02ak_fuzz_aesc_ref.log; tail -4 $O/r02ak_fuzz_aesc_ref.log
