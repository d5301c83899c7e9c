#!/bin/bash
# Round-2 closing measurements (one GPU): smoke, default bench, per-config
# bench, routed mix, reference arm, measured profile.
mkdir -p gpurun_out
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout -s KILL 1200 python bench.py --workload configs > gpurun_out/bench_configs.log 2>&1
timeout -s KILL 900 python bench.py --workload mix --mix-per-class 4 --decisions-out gpurun_out/mix_decisions.csv > gpurun_out/bench_mix.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout -s KILL 1500 python bench.py --workload profile --profile-out gpurun_out/b200_profile.json > gpurun_out/bench_profile.log 2>&1
echo done
