"""Attribute ncu's per-SASS-instruction counts to CUDA source lines.

    python tools/sass_lines.py <ncu source-page sass csv> <object or cubin> <mangled kernel name> [top]

The csv is `ncu -i <rep> --page source --csv --print-source sass` of one
launch (tools/ncu_source.sh); the object is the build/mrf_cuda/*.o the kernel
came from (compiled with -lineinfo). Line info comes from `nvdisasm -g`;
instruction offsets are matched by position from the kernel's first
instruction. Prints warp instructions executed and stall samples per source
line, largest first.
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
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
        cub = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
        txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    sec = txt.split(f".text.{kernel}")
    if len(sec) < 2:
        raise SystemExit(f"kernel {kernel} not in {obj}")
    body = f".text.{kernel}".join(sec[1:]).split("//--------------------- .text.")[0]
    cur = ("?", 0)
    table = {}
    for ln in body.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m:
            table[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return table


def main():
    csv_path, obj, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(io.StringIO(open(csv_path).read())))
    hdr = rows[1]
    ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > ie and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    table = line_table(obj, kernel)
    per = collections.defaultdict(lambda: [0, 0])
    total = 0
    for r in data:
        off = int(r[ia], 16) - base
        n = int(r[ie] or 0)
        s = int(r[iss] or 0)
        key = table.get(off, (("?", 0), ""))[0]
        per[key][0] += n
        per[key][1] += s
        total += n
    print(f"total warp instructions {total}")
    for (f, l), (n, s) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{n:12d} {100.0 * n / total:5.1f}%  stalls {s:7d}  {f}:{l}")


if __name__ == "__main__":
    main()
