timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | grep -E "passed|failed|^E " | head -20
timeout 1500 python -m pytest tests -x -q -m "slow and gpu" 2>&1 | grep -E "passed|failed|^E " | head -20
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/r01f_clocks.csv &
SMI=$!
timeout 600 python bench.py > gpurun_out/r01f_bench.json 2> gpurun_out/r01f_bench.err; echo bench rc=$?
kill $SMI
cat gpurun_out/r01f_bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|merge|fill|finalize" -c 20 --csv --log-file gpurun_out/r01f_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bf16 -s 1 -c 1 -o gpurun_out/r01f_attn python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu2 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bf16 -s 1 -c 1 -o gpurun_out/r01f_attn_d64 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --config c2d64 > /dev/null 2>&1; echo ncu3 rc=$?
