# round-2 GPU job 48: walk tests after the campaign_tables assertions
set -x
O=gpurun_out
python -m pytest tests/test_walks_gpu.py -m gpu -x -q -p no:cacheprovider > $O/r02av_pytest.log 2>&1; echo "rc=$?" >> $O/r02av_pytest.log; tail -3 $O/r02av_pytest.log
