"""Summarise an ncu report (or a --metrics gpu__time_duration launch-list CSV) into a committed
text table, and emit per-(layer, phase) DRAM traffic for bench.py's roofline.traffic field.

    python scripts/profile_summary.py full  gpurun_out/prof_C2.ncu-rep  profiles/r01_C2_full.txt  [layers.json]
    python scripts/profile_summary.py list  gpurun_out/launches_C2.csv  profiles/r01_C2_launches.txt
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__registers_per_thread", "sm__cycles_active.avg"]


def full(rep, out, phases_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    phases = json.load(open(phases_json)) if phases_json else None
    lines = [f"# ncu --set full summary of {rep}", "# one row per profiled launch; units from ncu",
             "# launch  kernel  time  dram_read  dram_write  tensor%  sm%  dram%  grid  regs  [layer.phase]"]
    traffic = {}
    for j, r in enumerate(data):
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
        vals = [r[idx[m]] for m in METRICS]
        u = [units[idx[m]] for m in METRICS]
        tag = ""
        if phases and j < len(phases):
            tag = phases[j]
            rd = float(r[idx["dram__bytes_read.sum"]]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[idx["dram__bytes_read.sum"]]]
            wr = float(r[idx["dram__bytes_write.sum"]]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[idx["dram__bytes_write.sum"]]]
            traffic[tag] = rd + wr
        lines.append(f"{j:3d}  {name:30s}  {vals[0]} {u[0]}  {vals[1]} {u[1]}  {vals[2]} {u[2]}  "
                     f"{float(vals[3]):.1f}  {float(vals[4]):.1f}  {float(vals[5]):.1f}  {vals[6]}  {vals[7]}  {tag}")
    open(out, "w").write("\n".join(lines) + "\n")
    return traffic


def launch_list(path, out):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list ({path})",
             "# cold-cache, serialised: compare SHARES, not absolutes", "# id  kernel  duration"]
    tot = 0.0
    recs = []
    for r in rows[1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[idx["Metric Value"]].replace(",", ""))
        recs.append((r[idx["ID"]], r[idx["Kernel Name"]].split("(")[0].replace("void ", ""), v, r[idx["Metric Unit"]]))
        tot += v
    for rid, k, v, u in recs:
        lines.append(f"{rid:>4s}  {k:40s}  {v:10.2f} {u}  share {v / tot * 100:5.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        t = full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
        if len(sys.argv) > 5:
            json.dump(t, open(sys.argv[5], "w"), indent=1)
    else:
        launch_list(sys.argv[2], sys.argv[3])
