"""Summarise ncu captures into profiles/ (development helper, run here after
gpurun brought the reports back).

  ncu_to_profile.py full <report.ncu-rep> <out.json> [cfg]
      per kernel launch: duration, dram read/write bytes (base units), issue
      active, warps active, fp64/tensor pipe use; for a matvec capture the
      dram bytes per matvec of the streamed passes (bench.py 'traffic')
  ncu_to_profile.py launches <launches.csv> <out.txt>
      per kernel name: launches, total time and share of the captured run
"""
import collections, csv, io, json, subprocess, sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def f(d, k):
    try:
        return float(d.get(k, "") or 0)
    except ValueError:
        return 0.0


KEYS = {"ms": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum",
        "dram_write": "dram__bytes_write.sum",
        "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dmma_pipe_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "l1_hit_pct": "l1tex__t_sector_hit_rate.pct", "l2_hit_pct": "lts__t_sector_hit_rate.pct",
        "registers": "launch__registers_per_thread"}


def full(rep, out_json):
    launches = []
    for d in raw(rep):
        e = {"kernel": d.get("Kernel Name", "")[:80]}
        for k, m in KEYS.items():
            e[k] = f(d, m)
        e["ms"] *= 1e-6  # ns -> ms in base units
        stalls = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""), f(d, h)) for h in d
            if h.startswith("smsp__average_warps_issue_stalled_") and
            h.endswith("_per_issue_active.ratio")), key=lambda x: -x[1])[:5]
        e["top_stalls"] = {k: round(v, 2) for k, v in stalls}
        launches.append(e)
    res = {"report": rep, "launches": launches}
    a = [e for e in launches if "hmv_warp_kernel" in e["kernel"]]
    if a:
        # pass A + pass B of one matvec = two consecutive hmv_warp_kernel launches
        per = sum(e["dram_read"] + e["dram_write"] for e in a) / (len(a) / 2)
        res["dram_bytes_per_matvec"] = per
        res["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of the streamed "
                       "passes (hmv_warp_kernel A + B) per matvec, ncu --set full "
                       "(cold-cache replay)")
    z = [e for e in launches if "hmv16_z_kernel" in e["kernel"]]
    y = [e for e in launches if "hmv16_y_kernel" in e["kernel"] or "hmv16_y2_kernel" in e["kernel"]]
    if z and y:
        # phase 1 + phase 2 of one 16-RHS pass
        per = (sum(e["dram_read"] + e["dram_write"] for e in z) / len(z) +
               sum(e["dram_read"] + e["dram_write"] for e in y) / len(y))
        res["dram_bytes_per_matvec"] = per
        res["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of hmv16_z_kernel + "
                       "hmv16_y(2)_kernel per 16-RHS pass, ncu --set full (cold-cache replay)")
    with open(out_json, "w") as fh:
        json.dump(res, fh, indent=1)
    for e in launches:
        print(f"{e['kernel'][:60]:60s} {e['ms']:8.3f} ms  dram {e['dram_read']/1e9:7.3f}+"
              f"{e['dram_write']/1e9:6.3f} GB  issue {e['issue_active_pct']:5.1f}%  "
              f"{e['top_stalls']}")
    if "dram_bytes_per_matvec" in res:
        print("dram bytes per matvec (A+B):", res["dram_bytes_per_matvec"])


def launches(csv_path, out_txt):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "ns"
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(unit, 1e-6)
        name = r[ki].split("(")[0][:70]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    with open(out_txt, "w") as fh:
        fh.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list\n"
                 f"# source: {csv_path}\n# kernel, launches, total ms, share of captured time\n")
        for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{name:70s} {n:6d} {ms:10.3f} {100 * ms / tot:6.2f}%\n")
    print(open(out_txt).read())


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3])
    else:
        launches(sys.argv[2], sys.argv[3])
