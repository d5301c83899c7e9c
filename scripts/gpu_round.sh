for i in 1 2 3 4 5; do timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -k "test_linear_formats_vs_oracle" > gpurun_out/kt_$i.log 2>&1; echo "EXIT $?" >> gpurun_out/kt_$i.log; done
