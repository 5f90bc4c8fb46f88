"""Print selected raw metrics per kernel from an .ncu-rep (diagnostic)."""
import csv, subprocess, sys
rep = sys.argv[1]
want = sys.argv[2].split(",") if len(sys.argv) > 2 else [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
    "sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
def col(name):
    for i, h in enumerate(hdr):
        if h == name or h.endswith("." + name) or h.split(".", 2)[-1] == name:
            return i
    return None
idx = {w: col(w) for w in want}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("npcg::", "")[:60]
    parts = []
    for w, i in idx.items():
        if i is None:
            continue
        parts.append("%s=%s%s" % (w.split("__")[-1][:40], r[i], units[i] if units[i] not in ("", "none") else ""))
    print(name)
    print("    " + "  ".join(parts))
