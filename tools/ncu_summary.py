"""Summarise ncu reports (gpurun_out/*.ncu-rep) into profiles/<round>_ncu_summary.json."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fmaheavy_pipe_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "inst_executed": "smsp__inst_executed.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
}


def unit_scale(unit: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "msecond": 1, "usecond": 1e-3,
            "nsecond": 1e-6, "us": 1e-3, "ns": 1e-6, "ms": 1, "s": 1e3, "second": 1e3}.get(unit, 1.0)


def summarise(rep: Path) -> list:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, m in KEYS.items():
            v = d.get(m)
            if v in (None, "", "n/a"):
                continue
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            if k.startswith("dram_") and k.endswith("bytes"):
                f *= unit_scale(u.get(m, "byte"))
            if k == "duration_ms":
                f *= unit_scale(u.get(m, "msecond"))
            rec[k] = f
        st = {}
        for m, v in d.items():
            if "average_warps_issue_stalled" in m and m.endswith("per_issue_active.ratio"):
                try:
                    st[m.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = float(v)
                except ValueError:
                    pass
        rec["top_stalls"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:5])
        res.append(rec)
    return res


if __name__ == "__main__":
    tag = sys.argv[1]
    reps = [Path(p) for p in sys.argv[2:]]
    allres = {r.stem: summarise(r) for r in reps}
    dst = Path("profiles") / f"{tag}_ncu_summary.json"
    dst.write_text(json.dumps(allres, indent=1))
    print(dst)
