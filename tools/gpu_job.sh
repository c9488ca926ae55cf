# round-2 GPU job 45: bench.py smoke after the roofline note (cfg2 without the AESC block, cfg1)
set -x
O=gpurun_out
python bench.py --no-aesc --steps 5 > $O/r02as_bench_cfg2.json 2> $O/r02as_bench_cfg2.err; echo "rc=$?"; python -c "
import json; d=json.loads(open('$O/r02as_bench_cfg2.json').read()); print(d['value'], d['roofline']['frac'], d['roofline'].get('note','')[:60])"
python bench.py --workload cfg1 --steps 5 > $O/r02as_bench_cfg1.json 2> $O/r02as_bench_cfg1.err; echo "rc=$?"; python -c "
import json; d=json.loads(open('$O/r02as_bench_cfg1.json').read()); print(d['value'], d['roofline']['frac'], d['roofline']['l2']['frac'])"
