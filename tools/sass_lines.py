"""Attribute the executed warp instructions of one profiled kernel to source lines.

    python tools/sass_lines.py <report.ncu-rep> <mangled kernel name> [top N]

Joins the per-instruction `Instructions Executed` column of `ncu --page source --csv` with the line table of
`nvdisasm -g` on the cubin inside paper_2505_22631_b200/liboscb.so (same build, -lineinfo): both list the kernel's
SASS in address order.  Prints the share of executed warp instructions per source line."""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def executed(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    return [(r[isrc].strip(), int(r[iex])) for r in rows[2:] if len(r) == len(hdr)]


def line_table(kernel):
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2505_22631_b200", "liboscb.so")], cwd=tmp,
                       capture_output=True)
        for cubin in glob.glob(os.path.join(tmp, "*.cubin")):
            text = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
            if ".text." + kernel not in text:
                continue
            seq, line, on = [], None, False
            for l in text.split("\n"):
                if ".section" in l[:12]:
                    on = (".text." + kernel) in l
                    continue
                if not on:
                    continue
                m = re.search(r'//## File "([^"]+)", line (\d+)', l)
                if m:
                    line = (os.path.basename(m.group(1)), int(m.group(2)))
                    continue
                if re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+.*?;", l):
                    seq.append(line)
            return seq
    raise SystemExit("kernel not found in liboscb.so")


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    ins, lines = executed(rep), line_table(kernel)
    if len(ins) != len(lines):
        raise SystemExit(f"instruction counts differ ({len(ins)} profiled, {len(lines)} disassembled): rebuild mismatch")
    per = collections.Counter()
    for (_, c), ln in zip(ins, lines):
        per[ln] += c
    total = sum(per.values())
    src = {}
    print(f"{total} warp instructions executed, {len(ins)} SASS instructions, {len(per)} source lines")
    for ln, c in per.most_common(top):
        text = ""
        if ln:
            if ln[0] not in src:
                found = glob.glob(os.path.join(ROOT, "paper_2505_22631_b200", "csrc", ln[0]))
                src[ln[0]] = open(found[0]).read().split("\n") if found else []
            if 0 < ln[1] <= len(src[ln[0]]):
                text = src[ln[0]][ln[1] - 1].strip()[:120]
        print(f"{100 * c / total:6.2f} %  {ln[0] if ln else '?'}:{ln[1] if ln else 0:<5d} {text}")


if __name__ == "__main__":
    main()
