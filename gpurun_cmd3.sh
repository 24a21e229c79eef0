set -x
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q -m "gpu and not slow" 2>&1 | tail -15
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r01_launches_bench.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bf16 -s 1 -c 1 -o gpurun_out/r01_attn python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r01_attn_ncu.log 2>&1; echo ncu2 rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:merge_kernel -c 1 -o gpurun_out/r01_merge python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r01_merge_ncu.log 2>&1; echo ncu3 rc=$?
ls -la gpurun_out
