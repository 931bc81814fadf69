"""Per-source-line instruction / stall shares of one kernel in an ncu report,
mapping SASS offsets to lines with nvdisasm -g of the built library
(development helper).
usage: ncu_src_lines.py <rep> <lib.so> <mangled-substr> [top] [launch-skip] [name-regex]"""
import collections, csv, io, os, re, subprocess, sys, tempfile
rep, lib, pat = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
fn = cur = None
ins = {}
for l in txt.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2))); continue
    if fn and pat in fn:
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m: ins[int(m.group(1), 16)] = cur
skip = sys.argv[5] if len(sys.argv) > 5 else "0"
kre = sys.argv[6] if len(sys.argv) > 6 else pat  # demangled-name regex for ncu
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + kre, "--launch-skip", skip,
                      "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
ie = hdr.index("Instructions Executed"); sm = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][0], 16)
by = collections.defaultdict(lambda: [0.0, 0.0])
for r in data:
    try: off = int(r[0], 16) - base
    except ValueError: continue
    c = ins.get(off)
    by[c][0] += float(r[ie] or 0); by[c][1] += float(r[sm] or 0)
ti = sum(v[0] for v in by.values()) or 1; ts = sum(v[1] for v in by.values()) or 1
src = {}
for c, v in sorted(by.items(), key=lambda kv: -kv[1][0])[:top]:
    s = ""
    if c:
        if c[0] not in src:
            try: src[c[0]] = open(c[0]).read().split("\n")
            except OSError: src[c[0]] = []
        s = src[c[0]][c[1] - 1].strip()[:78] if c[1] - 1 < len(src[c[0]]) else ""
    tag = f"{os.path.basename(c[0])}:{c[1]}" if c else "-"
    print(f"{tag:>26} inst {100*v[0]/ti:5.1f}% stall {100*v[1]/ts:5.1f}%  {s}")
