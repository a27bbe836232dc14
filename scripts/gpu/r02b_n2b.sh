# The N>1 bench path end to end with two gloo ranks sharing one GPU (exchange logic only; not a throughput), and the
# reference arm at N=2 (rank 0 alone runs it)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/n2b
KD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --tokens 8192 > gpurun_out/n2b/fkl.json 2> gpurun_out/n2b/fkl.err; echo "n2 fkl rc=$?"; tail -c 600 gpurun_out/n2b/fkl.json; tail -3 gpurun_out/n2b/fkl.err
KD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --config c3_jsd --tokens 8192 --no-variants > gpurun_out/n2b/jsd.json 2> gpurun_out/n2b/jsd.err; echo "n2 jsd rc=$?"; tail -c 400 gpurun_out/n2b/jsd.json; tail -3 gpurun_out/n2b/jsd.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/n2b/ref.json 2> gpurun_out/n2b/ref.err; echo "n2 ref rc=$?"; tail -c 300 gpurun_out/n2b/ref.json
