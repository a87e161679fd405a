"""Per-source-line instruction counts and stall samples of one profiled kernel.

    python scripts/sass_lines.py <report.ncu-rep> <object.o|.cubin> <kernel-substring> [launch#]

Joins `ncu --page source --print-source sass` (per-SASS counts) with the
line table of `nvdisasm -g` (needs -lineinfo builds)."""

import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def main():
    rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
    which = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    blocks = [b for b in blocks if kname in b["name"]]
    blk = blocks[which]
    hdr, data = blk["rows"][0], blk["rows"][1:]
    ia, ie, ist = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][ia], 16)
    cnt = {int(r[ia], 16) - base: (int(r[ie] or 0), int(r[ist] or 0)) for r in data}
    with tempfile.TemporaryDirectory() as td:
        cub = obj
        if obj.endswith(".o"):
            subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=td, capture_output=True)
            cub = str(next(Path(td).glob("*.cubin")))
        sass = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    # locate the kernel section: ".text.<mangled>:" label
    mangled = re.search(r"void (.*?)\(", blk["name"])
    lines, inside, line, src_file = {}, False, None, None
    for l in sass.split("\n"):
        if re.search(r"\.section\s+\.text\.", l):
            sec = l.split(".text.")[1].split(",")[0].strip().strip('"')
            inside = sec == target(blk["name"], sass)
            continue
        if not inside:
            continue
        m = re.search(r'//## File "(.*?)", line (\d+)', l)
        if m:
            src_file, line = m.group(1), int(m.group(2))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and line is not None:
            lines[int(m.group(1), 16)] = (src_file, line)
    agg, aggs = collections.Counter(), collections.Counter()
    for off, (c, s) in cnt.items():
        key = lines.get(off, ("?", -1))
        agg[key] += c
        aggs[key] += s
    tot, ts = sum(agg.values()) or 1, sum(aggs.values()) or 1
    print(f"{blk['name'][:120]}\n total warp-instructions {tot}")
    cache = {}
    for (f, ln), c in agg.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 30):
        text = ""
        if f != "?" and Path(f).name:
            p = Path(__file__).resolve().parent.parent / "paper_2306_12517_b200" / "csrc" / Path(f).name
            if p.exists():
                cache.setdefault(p, p.read_text().split("\n"))
                text = cache[p][ln - 1].strip()[:80]
        print(f"{c:>10} {100 * c / tot:5.1f}%  stall {100 * aggs[(f, ln)] / ts:5.1f}%  {Path(f).name}:{ln}  {text}")


_TARGET = None


def target(name, sass):
    global _TARGET
    if _TARGET is None:
        secs = re.findall(r'\.section\s+"?\.text\.(\S+?)"?,', sass)
        m = re.search(r"void bbx::image_kernel<(.*?)>\(", name)
        want = kernel_mangle_guess(name)
        _TARGET = next((s for s in secs if want and want in s), secs[0] if secs else "")
    return _TARGET


def kernel_mangle_guess(name):
    m = re.search(r"void bbx::(\w+)<(.*?)>\(", name)
    if not m:
        m = re.search(r"bbx::(\w+)\(", name)   # plain (non-template) kernel: _ZN3bbx<len><name>E...
        return f"{len(m.group(1))}{m.group(1)}E" if m else None
    fn, args = m.group(1), [a.strip() for a in m.group(2).split(",")]
    enc = []
    for a in args:
        if a in ("__half",):
            enc.append("6__half")
        elif a == "__nv_bfloat16":
            enc.append("13__nv_bfloat16")
        elif a == "float":
            enc.append("f")
        elif a in ("unsigned char", "uint8_t"):
            enc.append("h")
        else:
            mm = re.match(r"\((bool|int)\)(-?\d+)", a)
            if mm:
                enc.append(("Lb" if mm.group(1) == "bool" else "Li") + mm.group(2) + "E")
    return f"{len(fn)}{fn}I" + "".join(enc)


if __name__ == "__main__":
    main()
