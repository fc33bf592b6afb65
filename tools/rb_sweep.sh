# sweep env configurations of the bench (device legs only): det GB/s, q0 / q1 ms
for cfg in "$@"; do
  echo "== $cfg"; env $cfg python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['randomized']['q0']['ms_per_step'], d['randomized']['q1']['ms_per_step'])"
done
