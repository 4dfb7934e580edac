"""Joins an ncu SASS source page (csv) with nvdisasm --print-line-info output:
per CUDA source line -> instructions executed, warp-stall samples.
usage: sass_lines.py <ncu_sass.csv> <nvdisasm.sass> <mangled function> [file-substring]"""
import csv
import re
import sys
from collections import defaultdict


def line_map(path, fn, filesub):
    lines = open(path).read().split("\n")
    start = None
    for i, l in enumerate(lines):
        if l.startswith(".text." + fn + ":"):
            start = i
            break
    assert start is not None, fn
    cur = None
    m = {}
    inl = None
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith("\t.section") and m:
            break
        g = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
        if g:
            if "inlined at" in g.group(3):
                # keep the innermost location that lies in the target file
                pass
            if filesub in g.group(1):
                cur = int(g.group(2))
            continue
        g = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if g:
            m[int(g.group(1), 16)] = (cur, g.group(2).strip().rstrip(";"))
    return m


def main():
    csvp, sassp, fn = sys.argv[1:4]
    filesub = sys.argv[4] if len(sys.argv) > 4 else ".cu"
    rows = list(csv.reader(open(csvp)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ia, iex, istall, inis = hdr.index("Address"), hdr.index("Instructions Executed"), \
        hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Warp Stall Sampling (Not-issued Samples)")
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    base = int(data[0][ia], 16)
    lm = line_map(sassp, fn, filesub)
    per = defaultdict(lambda: [0, 0, 0, 0])
    tot_ex = tot_st = 0
    for r in data:
        off = int(r[ia], 16) - base
        ln, _ = lm.get(off, (None, ""))
        ex, st, ni = int(r[iex] or 0), int(r[istall] or 0), int(r[inis] or 0)
        p = per[ln]
        p[0] += ex; p[1] += st; p[2] += ni; p[3] += 1
        tot_ex += ex; tot_st += st
    print(f"total warp-instructions {tot_ex:,}  stall samples {tot_st:,}")
    print(f"{'line':>6} {'inst':>14} {'%inst':>6} {'samples':>9} {'%samp':>6} {'#sass':>6}")
    for ln, (ex, st, ni, n) in sorted(per.items(), key=lambda kv: -kv[1][0])[:60]:
        print(f"{str(ln):>6} {ex:>14,} {100 * ex / tot_ex:6.2f} {st:>9,} {100 * st / max(tot_st, 1):6.2f} {n:>6}")


if __name__ == "__main__":
    main()


def dump(csvp, sassp, fn, filesub, lo, hi):
    rows = list(csv.reader(open(csvp)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ia, iex, istall = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    base = int(data[0][ia], 16)
    lm = line_map(sassp, fn, filesub)
    for r in data:
        off = int(r[ia], 16) - base
        ln, ins = lm.get(off, (None, ""))
        if ln is not None and lo <= ln <= hi:
            print(f"{off:6x} {ln:5d} {int(r[iex] or 0):>12,} {int(r[istall] or 0):>6} {ins}")
