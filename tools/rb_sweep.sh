for cfg in "" "PSVD_TMA_NS=3" "PSVD_LA_NSUB=1" "PSVD_LA_NSUB=2" "PSVD_TMA_NS=4 PSVD_LA_NSUB=1"; do
  echo "== $cfg"; env $cfg python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['randomized']['q0']['ms_per_step'], d['randomized']['q1']['ms_per_step'])"
done
