timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | grep -E "passed|failed|^E " | head -20
for cfg in c2 c2d64; do
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --config $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg value %.1f  attn %.1f  clk %s %s' % (d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks']['reasons']))"
done
