for v in "" _poly0x00 _poly0x01 _poly0x11 _poly0x55; do
  for cfg in c2 c2d64; do
    CQS_LIB=$PWD/paper_2604_20819_b200/libcqs$v.so timeout 200 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --config $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $cfg value %.1f  attn %.1f  clk %s %s pw %s' % (d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['clocks'].get('power_w_max')))"
  done
done
