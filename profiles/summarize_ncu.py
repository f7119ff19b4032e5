"""Summarise an ncu --set full report into a small JSON/markdown table.

usage: python profiles/summarize_ncu.py <report.ncu-rep> [--json out.json] [--traffic out.json]
--traffic writes the per-launch DRAM traffic of the fused conv step launches
(bench.py's roofline.traffic).
Reads `ncu -i <rep> --page raw --csv` (ncu must be on PATH)."""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
}
SCALE = {"us": 1.0, "ns": 1e-3, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "Ghz": 1.0, "Mhz": 1e-3}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        e = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                e[k] = v * SCALE.get(units[i], 1.0)
        out.append(e)
    return out


if __name__ == "__main__":
    res = summarize(sys.argv[1])
    for e in res:
        print(json.dumps(e))
    if "--traffic" in sys.argv:
        step = [e for e in res if e["kernel"].startswith("k_rb_step")]
        n = max(len(step), 1)
        t = {"step_launches": len(step),
             "step_bytes_per_launch": sum(e["dram_read_bytes"] + e["dram_write_bytes"] for e in step) / n,
             "step_read_bytes_per_launch": sum(e["dram_read_bytes"] for e in step) / n,
             "step_write_bytes_per_launch": sum(e["dram_write_bytes"] for e in step) / n,
             "step_us_per_launch_cold": sum(e["time_us"] for e in step) / n,
             "source": sys.argv[1]}
        with open(sys.argv[sys.argv.index("--traffic") + 1], "w") as f:
            json.dump(t, f, indent=1)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
