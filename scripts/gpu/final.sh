# Round-end evidence: full GPU suite (parity log), default bench line, N=2 torchrun path (two gloo ranks sharing the
# one GPU: exercises the multi-rank bench code incl. the vocab-sharded and staged legs; not a throughput), launch list.
KD_PARITY_LOG=gpurun_out/parity.jsonl timeout 2000 python -m pytest tests -m gpu -q --tb=short > gpurun_out/gpu_full.log 2>&1; tail -3 gpurun_out/gpu_full.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 400 gpurun_out/bench_default.json
KD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_n2_gloo.json 2> gpurun_out/bench_n2_gloo.err; tail -c 600 gpurun_out/bench_n2_gloo.json; tail -3 gpurun_out/bench_n2_gloo.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches.csv
