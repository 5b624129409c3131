"""Copy a tools/round_bench.sh run (gpurun_out/round/) into profiles/: bench
lines, launch lists, backward timings, ncu key metrics of the cfg2 gather
kernel and the DRAM-traffic summary bench.py reads as roofline.traffic."""
import csv
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "round")
DST = os.path.join(ROOT, "profiles")
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}


def last_json(path):
    if not os.path.exists(path):
        return None
    lines = [x for x in open(path).read().splitlines() if x.startswith("{")]
    return lines[-1] if lines else None


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {k: {"value": x, "unit": u} for k, u, x in zip(r[0], r[1], r[2])}


def nbytes(m):
    return float(m["value"]) * SCALE[m["unit"]]


def update_ncu():
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
            "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
            "launch__registers_per_thread"]
    km_path = os.path.join(DST, "r1_ncu_key_metrics.json")
    km = json.load(open(km_path)) if os.path.exists(km_path) else {}
    summ_path = os.path.join(DST, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    # (capture, key-metrics entry, ncu_summary config, details csv)
    for cap, entry, cfg, details in [("cfg2_gather", "cfg2_gather_K2", "cfg2", "r1_cfg2_gather_ncu_details.csv"),
                                     ("cfg3_layer2_gather", "cfg3_layer2_gather_K2", "cfg3",
                                      "r1_cfg3_layer2_gather_ncu_details.csv"),
                                     ("cfg4_gather", "cfg4_gather_K3", "cfg4", "r1_cfg4_gather_ncu_details.csv")]:
        rep = os.path.join(SRC, cap + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        d = raw(rep)
        km[entry] = {k: d[k] for k in keys if k in d}
        km[entry]["kernel"] = d.get("Kernel Name", {}).get("value", "")
        m = km[entry]
        summ[cfg] = {"kernel": m["kernel"],
                     "dram_bytes_per_launch": nbytes(m["dram__bytes_read.sum"]) + nbytes(m["dram__bytes_write.sum"]),
                     "dram_read": nbytes(m["dram__bytes_read.sum"]), "dram_write": nbytes(m["dram__bytes_write.sum"]),
                     "source": "profiles/r1_ncu_key_metrics.json (ncu --set full --clock-control none)"}
        with open(os.path.join(DST, details), "w") as f:
            subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], stdout=f)
    json.dump(km, open(km_path, "w"), indent=1)
    json.dump(summ, open(summ_path, "w"), indent=1)


def main():
    import sys
    ncu_only = "--ncu-only" in sys.argv  # on the GPU box, between the captures and the bench lines
    update_ncu()
    if ncu_only:
        return
    for c in (1, 2, 3, 4, 5):
        line = last_json(os.path.join(SRC, f"bench_cfg{c}.json"))
        if line:
            open(os.path.join(DST, f"r1_bench_cfg{c}.json"), "w").write(line + "\n")
    line = last_json(os.path.join(SRC, "bench_reference_cfg2.json"))
    if line:
        open(os.path.join(DST, "r1_bench_reference_cfg2.json"), "w").write(line + "\n")
    for c in (2, 3, 4):
        p = os.path.join(SRC, f"launches_cfg{c}.csv")
        if os.path.exists(p):
            shutil.copy(p, os.path.join(DST, f"r1_cfg{c}_launches.csv"))
    bw = os.path.join(SRC, "bwd.jsonl")
    if os.path.exists(bw):
        shutil.copy(bw, os.path.join(DST, "r1_bench_backward.jsonl"))
    print("profiles updated")


if __name__ == "__main__":
    main()
