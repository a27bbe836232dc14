set -x
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv
for k in 64 16 4; do
  KD_KB_PER_ACC=$k timeout 900 python scripts/probe_parity_src.py c4 c2 > gpurun_out/probe_src_kb$k.log 2>&1
done
tail -n 30 gpurun_out/probe_src_kb*.log
