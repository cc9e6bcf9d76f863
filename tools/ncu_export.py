"""Export an .ncu-rep (run here, after gpurun brought it back) into profiles/: the details
page as text and the raw metrics of the first captured kernel as JSON (dev tool).

    python tools/ncu_export.py gpurun_out/prof_fused_cfg5.ncu-rep profiles/r02_ncu_full_fused_cfg5
"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
open(out + "_details.txt", "w").write(det)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: {"unit": u, "value": v} for h, u, v in zip(hdr, units, vals)}
json.dump(d, open(out + "_raw.json", "w"), indent=1, sort_keys=True)
def num(k):
    v = d[k]["value"].replace(",", "")
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d[k]["unit"], 1)
    return float(v) * mul
print(d.get("Kernel Name", {}).get("value"), "dram bytes", int(num("dram__bytes_read.sum") + num("dram__bytes_write.sum")),
      "duration", d["gpu__time_duration.sum"]["value"], d["gpu__time_duration.sum"]["unit"])
