# functional check of bench.py's multi-rank path (2 ranks, gloo, one GPU; NOT a timing)
PROHD_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config 2 --steps 2 --warmup 3 > gpurun_out/bench_mr.json 2> gpurun_out/bench_mr.err; echo "rc=$?" >> gpurun_out/bench_mr.err
