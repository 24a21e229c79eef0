timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | grep -E "passed|failed|Error|error|^E " | head -20
timeout 300 python -m pytest tests/test_gpu_stream.py -q -m "gpu and not slow" 2>&1 | grep -E "^E |passed|failed" | head -20
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -1
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --config c2d64 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"merge|fill|finalize" -c 4 --csv --log-file gpurun_out/r01d_merge.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu rc=$?
