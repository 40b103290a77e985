"""Summarise ncu --set full reports into profiles/ncu_traffic.json (the source
of bench.py's roofline.traffic and roofline.limiter).

usage: python tools/ncu_summary.py OUT.json KEY=report.ncu-rep[:kernel-substring[:units]] ...
Per key: the first launch in the report whose name contains the substring;
units (numbers or samples the launch processed) adds inst_per_unit = warp
instructions executed per unit (the bench's issue roofline)."""
import csv
import io
import json
import subprocess
import sys

M = {"gpu__time_duration.sum": "duration_ms_ncu", "dram__bytes_read.sum": "dram_bytes_read",
     "dram__bytes_write.sum": "dram_bytes_write",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
     "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active": "fmaheavy_pipe_pct",
     "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed": "fmaheavy_pipe_pct_elapsed",
     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
     "smsp__inst_executed.sum": "inst_executed",
     "sm__cycles_active.avg": "sm_cycles_active",
     "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
     "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
     "launch__registers_per_thread": "registers", "launch__grid_size": "grid",
     "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct"}
UNIT = {"dram__bytes_read.sum": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
        "gpu__time_duration.sum": {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}}
UNIT["dram__bytes_write.sum"] = UNIT["dram__bytes_read.sum"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    return [(dict(zip(hdr, x)), dict(zip(hdr, units))) for x in r[2:]]


def main():
    out, specs = sys.argv[1], sys.argv[2:]
    res = {}
    for sp in specs:
        key, rest = sp.split("=", 1)
        rep, _, sub = rest.partition(":")
        sub, _, units = sub.partition(":")
        for d, u in rows(rep):
            if sub and sub not in d["Kernel Name"]:
                continue
            e = {"kernel": d["Kernel Name"]}
            for m, k in M.items():
                v = d.get(m, "")
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                x *= UNIT.get(m, {}).get(u.get(m, ""), 1.0)
                e[k] = x
            if "fmaheavy_pipe_pct" not in e and "fmaheavy_pipe_pct_elapsed" in e:
                e["fmaheavy_pipe_pct"] = e["fmaheavy_pipe_pct_elapsed"]
            if units and e.get("inst_executed"):
                e["units"] = float(units)
                e["inst_per_unit"] = e["inst_executed"] / float(units)
            e["source"] = f"ncu --set full --clock-control none ({rep})"
            res[key] = e
            break
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
