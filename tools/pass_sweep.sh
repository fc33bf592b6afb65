#!/bin/bash
# la / projB durations of the pipelined randomized stream (config 2, q = 0) under env variants
# (arguments: extra variants, e.g. "PSVD_TMA_NS=2"; a leading "-" skips the default set)
if [ "$1" == "-" ]; then shift; set -- "" "$@"; else set -- "" "PSVD_TMA_NS=2" "PSVD_GRAM_DBG=1" "$@"; fi
for v in "$@"; do
  echo "== ${v:-default}"
  env $v timeout 120 python tools/rand_trace.py 0 2>&1 >/dev/null | python tools/trace_passes.py
done
