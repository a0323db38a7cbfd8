bash tools/exp/kb.sh
python bench.py --no-cpu --steps 40 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],3), d['clocks'], round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['column_kernel']['avg_launch_ms'],4))"
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
