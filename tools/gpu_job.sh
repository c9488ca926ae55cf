# round-2 GPU job 44: bench.py --gpus 2 --dist-backend gloo under torch.distributed.run (two ranks sharing the GPU), final build
set -x
O=gpurun_out
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dist-backend gloo --workload cfg1 --steps 5 --warmup 3 > $O/r02ar_bench_gloo2_cfg1.json 2> $O/r02ar_gloo2_cfg1.err; tail -c 600 $O/r02ar_bench_gloo2_cfg1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --dist-backend gloo --workload cfg3 > $O/r02ar_bench_gloo2_cfg3.json 2> $O/r02ar_gloo2_cfg3.err; tail -c 600 $O/r02ar_bench_gloo2_cfg3.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 --no-aesc > $O/r02ar_bench_gloo2_cfg2.json 2> $O/r02ar_gloo2_cfg2.err; tail -c 600 $O/r02ar_bench_gloo2_cfg2.json
