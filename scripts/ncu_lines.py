"""Map ncu SASS-level stall samples (--page source --csv --print-source sass) to CUDA source lines
using `nvdisasm -g` line info of the same cubin. Usage: ncu_lines.py sass.csv disasm.txt kernel_substr"""
import csv
import re
import sys
from collections import defaultdict


def main(sass_csv, dis_txt, kname, top=45):
    rows = list(csv.reader(open(sass_csv)))
    h = rows[1]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > i_s]
    base = int(data[0][0], 16)
    samples = {int(r[0], 16) - base: int(r[i_s]) if r[i_s].isdigit() else 0 for r in data}
    # offsets -> line from nvdisasm -g
    lines = {}
    infn, cur = False, None
    for ln in open(dis_txt):
        if ".text." in ln and kname in ln and ln.strip().startswith(".section"):
            infn = True
            continue
        if infn and ln.strip().startswith(".section"):
            break
        if not infn:
            continue
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if "//##" in ln and m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        m2 = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
        if m2 and cur is not None:
            lines[int(m2.group(1), 16)] = cur
    agg = defaultdict(int)
    for off, n in samples.items():
        agg[lines.get(off, ("?", 0))] += n
    tot = sum(agg.values())
    srcdir = sys.argv[4] if len(sys.argv) > 4 else None
    cache = {}
    for (f, line), n in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        txt = ""
        if srcdir and line > 0:
            if f not in cache:
                try:
                    cache[f] = open(f"{srcdir}/{f}").read().splitlines()
                except OSError:
                    cache[f] = []
            if line <= len(cache[f]):
                txt = cache[f][line - 1].strip()[:80]
        print(f"{f[:10]:>10}:{line:<5d} {n:7d} {100 * n / tot:5.1f}%  {txt}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
