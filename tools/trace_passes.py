"""Mean durations of the traced segments of the last run of tools/rand_trace.py (stderr on stdin):
la (look-ahead sketch, low-priority stream) and projB (projection pass) per update."""
import re, sys, collections
runs, cur = [], None
for line in sys.stdin:
    if line.startswith("---- run"):
        cur = []
        runs.append(cur)
    m = re.match(r"psvd_trace (\S+)\s+([-\d.]+) ms", line)
    if m and cur is not None:
        cur.append((re.sub(r"\[\d+\]$", "", m.group(1)), float(m.group(2))))
last = runs[-1]
t = collections.defaultdict(list)
for name, v in last:
    t[name].append(v)
def span(a, b):
    xs = [y - x for x, y in zip(t.get(a, []), t.get(b, []))]
    return sum(xs) / len(xs) if xs else float("nan"), len(xs)
for a, b in [("lo:la_begin", "lo:la_end"), ("hi:projB", "hi:projB_end")]:
    m, n = span(a, b)
    print(f"{a}->{b}: {m:.3f} ms (n={n})")
print("total", last[-1][1] if last else None, "ms")
