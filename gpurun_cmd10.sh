timeout 300 python tools_debug_gpu.py 2>&1 | tail -12
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | grep -E "passed|failed|^E " | head -20
for v in "" _onecta; do
CQS_LIB=$PWD/paper_2604_20819_b200/libcqs$v.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v value %.1f  attn %.1f  clk %s %s' % (d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks']['reasons']))"
done
