mkdir -p gpurun_out/ab
timeout 600 python tools/walk_probe.py cfg4 500 18944 > gpurun_out/ab/probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > gpurun_out/ab/pytest.log 2>&1; echo rc=$? >> gpurun_out/ab/pytest.log
timeout 600 python bench.py --force-dist --steps 2 --warmup 1 --no-extras --no-cpu-baseline --parity-chains 0 > gpurun_out/ab/dist.json 2> gpurun_out/ab/dist.err
cat gpurun_out/ab/probe.log; tail -2 gpurun_out/ab/pytest.log; head -c 400 gpurun_out/ab/dist.json; tail -3 gpurun_out/ab/dist.err
