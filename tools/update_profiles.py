"""Copy a tools/round_bench.sh run (gpurun_out/round_$R/) into profiles/ as
${R}_*: bench lines, launch lists, backward timings, ncu key metrics of the
captured kernels and the DRAM-traffic summary bench.py reads as
roofline.traffic (profiles/ncu_summary.json)."""
import csv
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = os.environ.get("R", "r2")
SRC = os.path.join(ROOT, "gpurun_out", "round_" + R)
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
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
            "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
            "launch__registers_per_thread"]
    km_path = os.path.join(DST, f"{R}_ncu_key_metrics.json")
    km = json.load(open(km_path)) if os.path.exists(km_path) else {}
    summ_path = os.path.join(DST, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    # (capture, key-metrics entry, ncu_summary config or None)
    for cap, entry, cfg in [("cfg2_gather", "cfg2_gather_K2", "cfg2"),
                            ("cfg3_layer2_gather", "cfg3_layer2_gather_K2", "cfg3"),
                            ("cfg3_head", "cfg3_head_narrow", None),
                            ("cfg4_gather", "cfg4_gather_K3_pixel", "cfg4"),
                            ("cfg1_gather", "cfg1_gather", "cfg1"),
                            ("cfg5_gather", "cfg5_shard_gather", "cfg5"),
                            ("cfg6_gather", "cfg6_conv_stage2_gather", "cfg6"),
                            ("cfg7_gather", "cfg7_conv_stage3_gather", "cfg7")]:
        rep = os.path.join(SRC, cap + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        d = raw(rep)
        km[entry] = {k: d[k] for k in keys if k in d}
        km[entry]["kernel"] = d.get("Kernel Name", {}).get("value", "")
        m = km[entry]
        if cfg:
            summ[cfg] = {"kernel": m["kernel"],
                         "dram_bytes_per_launch": nbytes(m["dram__bytes_read.sum"]) + nbytes(m["dram__bytes_write.sum"]),
                         "dram_read": nbytes(m["dram__bytes_read.sum"]), "dram_write": nbytes(m["dram__bytes_write.sum"]),
                         "source": f"profiles/{R}_ncu_key_metrics.json (ncu --set full --clock-control none)"}
        with open(os.path.join(DST, f"{R}_{cap}_ncu_details.csv"), "w") as f:
            subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], stdout=f)
    json.dump(km, open(km_path, "w"), indent=1)
    json.dump(summ, open(summ_path, "w"), indent=1)


def main():
    import sys
    ncu_only = "--ncu-only" in sys.argv  # on the GPU box, between the captures and the bench lines
    if ncu_only:
        update_ncu()
        return
    # here: the box's extracted ncu files (round_bench.sh copies them to $SRC/prof)
    prof = os.path.join(SRC, "prof")
    if os.path.isdir(prof):
        for f in os.listdir(prof):
            shutil.copy(os.path.join(prof, f), os.path.join(DST, f))
    update_ncu()  # no-op unless .ncu-rep files are present locally
    for name in ([f"bench_cfg{c}" for c in (1, 2, 3, 4, 5, 6, 7)] + ["bench_cfg2_exact"] +
                 [f"bench_reference_cfg{c}" for c in (1, 2, 3, 4, 6, 7)]):
        line = last_json(os.path.join(SRC, name + ".json"))
        if line:
            open(os.path.join(DST, f"{R}_{name}.json"), "w").write(line + "\n")
    for c in (1, 2, 3, 4, 5, 6, 7):
        p = os.path.join(SRC, f"launches_cfg{c}.csv")
        if os.path.exists(p):
            shutil.copy(p, os.path.join(DST, f"{R}_cfg{c}_launches.csv"))
    bw = os.path.join(SRC, "bwd.jsonl")
    if os.path.exists(bw):
        shutil.copy(bw, os.path.join(DST, f"{R}_bench_backward.jsonl"))
    print("profiles updated")


if __name__ == "__main__":
    main()
