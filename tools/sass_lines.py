"""Attribute ncu per-SASS-instruction stall samples to CUDA source lines.

usage: python tools/sass_lines.py REPORT.ncu-rep OBJECT.o KERNEL_MANGLED [top]

Joins `ncu --page source --print-source sass` (per-address samples) with the
line table `nvdisasm --print-line-info` prints for the kernel's cubin (the
object must be the one the profiled library was linked from, built with
-lineinfo). Prints the top source lines by stall samples and a per-file total.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
                   capture_output=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cubin)],
                         capture_output=True, text=True).stdout
    start = dis.find(f".text.{kernel}:")  # cut the kernel's own section
    dis = dis[start:] if start >= 0 else dis
    nxt = dis.find("//---------------------", 10)
    dis = dis[:nxt] if nxt > 0 else dis
    cur = None
    table = {}
    for ln in dis.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            if cur is None or "inlined at" not in ln:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            table[int(m.group(1), 16)] = cur
    return table


def samples(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    body = "\n".join(lines[1:])  # first line: kernel name
    rows = csv.DictReader(io.StringIO(body))
    res = []
    for r in rows:
        try:
            addr = int(r["Address"], 16)
            s = int(r["Warp Stall Sampling (All Samples)"] or 0)
            ex = int(r.get("Instructions Executed") or 0)
        except (KeyError, ValueError):
            continue
        res.append((addr, s, r["Source"], ex))
    base = min(r[0] for r in res) if res else 0  # runtime addresses -> section offsets
    return [(a - base, s, src, ex) for a, s, src, ex in res]


def main():
    rep, obj, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    table = line_table(obj, kernel)
    per_line = collections.Counter()
    per_file = collections.Counter()
    inst_line = collections.Counter()
    total = 0
    tinst = 0
    for addr, s, _, ex in samples(rep):
        total += s
        tinst += ex
        key = table.get(addr, ("?", 0))
        per_line[key] += s
        per_file[key[0]] += s
        inst_line[key] += ex
    src_cache = {}
    root = os.path.dirname(os.path.abspath(obj))
    csrc = os.path.join(os.path.dirname(root), "paper_2410_18944_b200", "csrc")
    for (f, n), s in per_line.most_common(top):
        if f not in src_cache:
            p = os.path.join(csrc, f)
            src_cache[f] = open(p).read().splitlines() if os.path.exists(p) else []
        text = src_cache[f][n - 1].strip() if 0 < n <= len(src_cache[f]) else ""
        print(f"{100.0 * s / max(total, 1):5.1f}%  {f}:{n}  {text[:90]}")
    print("-- top lines by executed warp instructions")
    for (f, n), c in inst_line.most_common(top // 2):
        if f not in src_cache:
            p = os.path.join(csrc, f)
            src_cache[f] = open(p).read().splitlines() if os.path.exists(p) else []
        text = src_cache[f][n - 1].strip() if 0 < n <= len(src_cache[f]) else ""
        print(f"{100.0 * c / max(tinst, 1):5.1f}%  {f}:{n}  {text[:90]}")
    print("-- per file")
    for f, s in per_file.most_common():
        print(f"{100.0 * s / max(total, 1):5.1f}%  {f}")


if __name__ == "__main__":
    main()
