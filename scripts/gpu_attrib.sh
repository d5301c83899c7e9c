mkdir -p gpurun_out
bash scripts/step_attrib.sh 2
timeout -s KILL 300 python scripts/attn_timeline.py 2 200 > gpurun_out/attn_tl.txt 2>&1
timeout -s KILL 300 python scripts/attn_timeline.py 2 129 > gpurun_out/attn_tl129.txt 2>&1
