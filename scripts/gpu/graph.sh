timeout 600 python -m pytest tests/test_gpu_graph.py -q --tb=short > gpurun_out/graph_tests.log 2>&1; tail -15 gpurun_out/graph_tests.log
timeout 600 python bench.py --graph --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err; tail -3 gpurun_out/bench_graph.err
python -c "import json; d=json.loads(open('gpurun_out/bench_graph.json').read().strip().splitlines()[-1]); print(round(d['value']), d['ms_per_step'], d['cuda_graph'])"
timeout 600 python bench.py --graph --tokens 2048 --steps 50 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_graph_small.json 2> gpurun_out/bench_graph_small.err; tail -3 gpurun_out/bench_graph_small.err
python -c "import json; d=json.loads(open('gpurun_out/bench_graph_small.json').read().strip().splitlines()[-1]); print(round(d['value']), d['ms_per_step'], d['cuda_graph'])"
