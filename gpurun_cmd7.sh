for v in "" _mufu _poly4 _noexp _nosoftmax; do
  for cfg in c2 c2d64; do
    echo "variant=$v cfg=$cfg"
    CQS_LIB=$PWD/paper_2604_20819_b200/libcqs$v.so timeout 200 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --config $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' value %.1f  attn %.1f  clk %s %s' % (d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks']['reasons']))"
  done
done
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q 2>&1 | grep -E "passed|failed|^E " | head
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1
