#!/bin/bash
# Round-2 closing measurements after the decode latency work (one GPU):
# default bench, per-config bench, routed mix, reference arm, ncu launch list
# of one W4 decode step, ncu --set full of the decode attention and the W4
# qkv GEMV, in-graph step attribution, measured profile.
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout -s KILL 1200 python bench.py --workload configs > gpurun_out/bench_configs.log 2>&1
timeout -s KILL 900 python bench.py --workload mix --mix-per-class 4 --decisions-out gpurun_out/mix_decisions.csv > gpurun_out/bench_mix.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w4.csv python scripts/decode_once.py --mode 2 --new 4 > gpurun_out/ncu_l.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 40 -c 1 -o gpurun_out/attn_dec_r02 python scripts/decode_once.py --mode 2 --new 4 --graphs 0 > gpurun_out/ncu_a.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:gemv_w4 -s 3 -c 1 -o gpurun_out/w4_qkv_r02 python scripts/gemv_micro.py 2 qkv > gpurun_out/ncu_q.log 2>&1
bash scripts/step_attrib.sh 2
timeout -s KILL 1500 python bench.py --workload profile --profile-out gpurun_out/b200_profile.json > gpurun_out/bench_profile.log 2>&1
echo done
