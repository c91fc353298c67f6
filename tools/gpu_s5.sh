#!/bin/bash
# GPU suite + smoke + C5 bench line + default (C3) bench line
O=gpurun_out/${1:-s5}; mkdir -p $O
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-sweep > $O/bench_c5.json 2> $O/bench_c5.err; echo "rc=$?" >> $O/bench_c5.err
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
