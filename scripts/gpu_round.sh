timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout -s KILL 900 python bench.py --workload configs > gpurun_out/bench_configs.log 2>&1
timeout -s KILL 900 python bench.py --workload mix --mix-per-class 4 --decisions-out gpurun_out/mix_decisions.csv > gpurun_out/bench_mix.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout -s KILL 1200 python bench.py --workload profile --profile-out gpurun_out/b200_profile.json > gpurun_out/bench_profile.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w4.csv python scripts/decode_once.py --mode 2 --new 4 > gpurun_out/ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 40 -c 1 -o gpurun_out/attn_dec3 python scripts/decode_once.py --mode 2 --new 4 --graphs 0 > gpurun_out/ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemv_w4 -s 3 -c 1 -o gpurun_out/w4_gu python scripts/gemv_micro.py 2 gate_up > gpurun_out/ncu1.log 2>&1
timeout -s KILL 300 python scripts/gemv_micro.py 2,1,0 > gpurun_out/gemv_micro_all.txt 2>&1
timeout -s KILL 300 python scripts/attn_timeline.py 2 200 > gpurun_out/attn_tl.txt 2>&1
