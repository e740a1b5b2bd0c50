# functional check of bench.py's multi-rank path (2 ranks, gloo, ONE GPU shared: NOT a timing)
CFG=${CFG:-2}
PROHD_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config $CFG --steps 1 --warmup 3 > gpurun_out/bench_mr.json 2> gpurun_out/bench_mr.err; echo "rc=$?" >> gpurun_out/bench_mr.err
