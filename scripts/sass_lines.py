"""Static SASS instruction count per source line for one kernel (development helper).
usage: sass_lines.py <lib.so> <kernel-name-substring> [top]"""
import collections, os, re, subprocess, sys, tempfile
lib, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = txt.split("\n")
cur, fn, counts, total = None, None, collections.Counter(), 0
src = {}
for l in lines:
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    if fn and pat in fn and re.search(r"/\*[0-9a-f]{4,}\*/", l):
        counts[cur] += 1
        total += 1
print("total", total)
for (f, ln), c in counts.most_common(top):
    if f not in src:
        try: src[f] = open(f).read().split("\n")
        except OSError: src[f] = []
    s = src[f][ln - 1].strip()[:80] if ln - 1 < len(src[f]) else ""
    print(f"{c:5d} {os.path.basename(f)}:{ln} {s}")
