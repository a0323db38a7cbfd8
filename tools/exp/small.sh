for b in 8 16; do for mx in 0 1; do
  BP_MIXED=$mx python bench.py --no-cpu --batch $b --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch $b mixed $mx', round(d['value'],3), d['clocks']['sm_mhz'], d['clocks']['power_w'])"
done; done
