mkdir -p gpurun_out/q9
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "build or pcg or c2" > gpurun_out/q9/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q9/pytest.log
python tools/phases.py C2 > gpurun_out/q9/c2.json 2>&1
timeout 600 python tools/phases.py C5 > gpurun_out/q9/c5.json 2>&1
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/q9/bench.json 2> gpurun_out/q9/bench.err
