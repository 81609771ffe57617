"""Build profiles/ncu_summary.json from `ncu --set full` reports (profiling helper, not product
code).  usage: ncu_summary.py OUT.json name=REPORT.ncu-rep[:label] ...

For every report: the key metrics of its (single) captured launch, DRAM bytes per launch and
the warp-stall reasons per issued instruction."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active", "launch__grid_size",
    "launch__block_size",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def summarise(rep):
    r = raw(rep)
    m = {k: list(r[k]) for k in KEYS if k in r}
    stalls = {}
    issued = float(r["smsp__inst_executed.sum"][0].replace(",", ""))
    for k, (v, _) in r.items():
        pre = "smsp__pcsamp_warps_issue_stalled_"
        if k.startswith(pre) and not k.endswith("_not_issued"):
            try:
                stalls[k[len(pre):]] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values())
    sel = stalls.get("selected", 0.0) or 1.0
    m["stalls_per_issue"] = {k: round(v / sel, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])
                             if v / sel >= 0.05} if tot else {}
    rd = float(r["dram__bytes_read.sum"][0].replace(",", "")) * UNIT.get(r["dram__bytes_read.sum"][1], 1)
    wr = float(r["dram__bytes_write.sum"][0].replace(",", "")) * UNIT.get(r["dram__bytes_write.sum"][1], 1)
    name = r.get("Kernel Name", r.get("Function Name", ("?", "")))[0]
    return {"name": name, "dram_bytes_per_launch": rd + wr, "instructions_per_launch": issued, "metrics": m}


def main():
    out = sys.argv[1]
    res = {"round": 2, "gpu": "NVIDIA B200 (sm_100a)",
           "how": "ncu --set full --clock-control none --import-source on -k regex:<kernel> -s <skip> -c 1 "
                  "python bench.py --steps 1 --warmup 3 --no-cpu-baseline (one launch, replayed)",
           "kernels": {}}
    for arg in sys.argv[2:]:
        key, spec = arg.split("=", 1)
        rep, _, label = spec.partition(":")
        res["kernels"][key] = summarise(rep)
        if label:
            res["kernels"][key]["workload"] = label
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: (v["name"][:60], v["metrics"]["gpu__time_duration.sum"]) for k, v in res["kernels"].items()}))


if __name__ == "__main__":
    main()
