timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -8
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|merge|fill" -c 20 --csv --log-file gpurun_out/r01b_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bf16 -s 1 -c 1 -o gpurun_out/r01b_attn python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu2 rc=$?
