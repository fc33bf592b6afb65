"""Attribute an ncu SASS source page (csv) to CUDA source lines via nvdisasm -g line info."""
import collections, csv, re, subprocess, sys

def line_map(cubin, func):
    out = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
    m, cur, on = {}, None, False
    for ln in out.splitlines():
        if ln.startswith(".text."):
            on = ln.startswith(".text." + func)
            continue
        if not on:
            continue
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = (g.group(1).split("/")[-1], int(g.group(2)))
            continue
        g = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if g:
            m[int(g.group(1), 16)] = cur
    return m

def main(csvf, cubin, func, top=40):
    rows = list(csv.reader(open(csvf)))
    hdr = rows[1]
    ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) >= len(hdr) and re.fullmatch(r"(0x)?[0-9a-fA-F]+", r[ia])]
    end = next((i for i in range(1, len(data)) if int(data[i][ia], 16) < int(data[i - 1][ia], 16)), len(data))
    data = data[:end]  # first kernel only
    start = int(data[0][ia], 16)
    lm = line_map(cubin, func)
    agg = collections.defaultdict(lambda: [0, 0])
    for r in data:
        off = int(r[ia], 16) - start
        key = lm.get(off, ("?", -1))
        agg[key][0] += int(r[ie]); agg[key][1] += int(r[iss])
    src = {}
    tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
    print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
    for (f, l), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        try:
            text = open(f"paper_2108_08845_b200/csrc/{f}").read().splitlines()[l - 1].strip()[:80]
        except Exception:
            text = ""
        print(f"{f}:{l:4d} inst {i:9d} ({100*i/tot_i:5.1f}%) samples {s:5d} ({100*s/tot_s:5.1f}%)  {text}")

if __name__ == "__main__":
    main(*sys.argv[1:4])
