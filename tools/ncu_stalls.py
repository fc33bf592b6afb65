"""Per-source-line stall-reason breakdown of an ncu source page (csv): tools/ncu_lines.py with the
stall_* columns.  usage: ncu_stalls.py page.csv cubin mangled_function_prefix [top]"""
import collections, csv, re, sys
sys.path.insert(0, "tools")
from ncu_lines import line_map

def main(csvf, cubin, func, top=30):
    rows = list(csv.reader(open(csvf)))
    hdr = rows[1]
    ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    isrc = hdr.index("Source")
    st = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = [r for r in rows[2:] if len(r) >= len(hdr) and re.fullmatch(r"(0x)?[0-9a-fA-F]+", r[ia])]
    start = int(data[0][ia], 16)
    lm = line_map(cubin, func)
    agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), collections.Counter()])
    for r in data:
        off = int(r[ia], 16) - start
        key = lm.get(off, ("?", -1))
        a = agg[key]
        a[0] += int(r[ie]); a[1] += int(r[iss])
        for i, h in st:
            if r[i] not in ("", "0"):
                a[2][h[6:]] += int(r[i])
        a[3][r[isrc].split()[0] if r[isrc] else "?"] += int(r[iss])
    tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
    allst = collections.Counter()
    for v in agg.values():
        allst.update(v[2])
    print(f"total warp-instructions {tot_i}, stall samples {tot_s}; by reason: " +
          ", ".join(f"{k} {100*v/tot_s:.1f}%" for k, v in allst.most_common(8)))
    for (f, l), (i, s, c, ops) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(top)]:
        try:
            text = open(f"paper_2108_08845_b200/csrc/{f}").read().splitlines()[l - 1].strip()[:60]
        except Exception:
            text = ""
        why = " ".join(f"{k}:{100*v/max(s,1):.0f}" for k, v in c.most_common(3))
        op = ",".join(k for k, _ in ops.most_common(2))
        print(f"{f}:{l:4d} inst {100*i/tot_i:5.1f}% smp {100*s/tot_s:5.1f}% [{why}] {op} | {text}")

if __name__ == "__main__":
    main(*sys.argv[1:5])
