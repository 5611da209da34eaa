"""Summarise the round-2 ncu captures (gpurun_out/r02_ncu_*.ncu-rep) into small JSON files
under profiles/ (the .ncu-rep files themselves are too large to keep): per kernel the
duration, DRAM bytes, tensor-pipe / DRAM / issue utilisation, registers, and the warp-stall
reasons summed over the kernel; plus profiles/r02_ncu_traffic.json (DRAM bytes per launch,
the `traffic` bench.py reports) and the per-kernel shares of the launch lists."""
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
OUT = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "sm__cycles_elapsed.avg", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
# bench.py traffic keys of the captured launches
TRAFFIC = {"r02_ncu_l1_3x3_U": "r50_64_64_56_3x3s1_U", "r02_ncu_l1_3x3_F": "r50_64_64_56_3x3s1_F",
           "r02_ncu_l3_3x3_F": "r50_256_256_14_3x3s1_F", "r02_ncu_l3_1x1_F": "r50_1024_256_14_1x1s1_F",
           "r02_ncu_l3_1x1_U": "r50_256_1024_14_1x1s1_U", "r02_ncu_cfg2_U": "cfg2_U",
           "r02_ncu_l1_1x1_res_F": "r50_64_256_56_1x1s1_F", "r02_ncu_l4_3x3_U": "r50_512_512_7_3x3s1_U",
           "r02_ncu_l4_3x3_F": "r50_512_512_7_3x3s1_F", "r02_ncu_l4_1x1_F": "r50_2048_512_7_1x1s1_F"}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "").split("(")[0].replace("void ", "")}
        for key in KEYS:
            if key in d and d[key] != "":
                try:
                    k[key] = float(d[key].replace(",", ""))
                    if u.get(key):
                        k[key + " [unit]"] = u[key]
                except ValueError:
                    pass
        st = {h: float(d[h].replace(",", "")) for h in hdr
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and d.get(h, "") not in ("", "n/a")
              and not h.endswith("_not_issued")}
        tot = sum(st.values()) or 1.0
        k["stall_share_top"] = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(v / tot, 3)
                                for h, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]}
        kernels.append(k)
    return kernels


def bytes_of(k):
    def b(key):
        v = k.get(key)
        unit = k.get(key + " [unit]", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        return v * scale if v is not None else None
    r, w = b("dram__bytes_read.sum"), b("dram__bytes_write.sum")
    return (r or 0) + (w or 0) if r is not None else None


def launches(path, out, note):
    rows = list(csv.reader(open(path)))
    hdr, ks = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(d.get("Metric Unit", "nsecond"), 1.0)
                ks.append((d["Kernel Name"].split("(")[0].replace("void ", ""), float(d["Metric Value"].replace(",", "")) * scale))
    agg = {}
    for n, t in ks:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values()) or 1.0
    with open(out, "w") as f:
        f.write(f"# {note}\n# ncu --metrics gpu__time_duration.sum --clock-control none: serialised and cold-cache,\n"
                "# compare SHARES with the bench's live CUDA-event kernel times\nkernel,launches,total_ns,share\n")
        for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{n},{c},{int(t)},{t / tot:.4f}\n")


def main(src):
    # merged into the committed summaries (a capture set may cover only some kernels)
    summary, traffic = {}, {}
    try:
        summary = json.load(open(os.path.join(OUT, "r02_ncu_full.json")))["captures"]
        traffic = json.load(open(os.path.join(OUT, "r02_ncu_traffic.json")))
    except (OSError, ValueError, KeyError):
        pass
    for rep in sorted(glob.glob(os.path.join(src, "r02_ncu_*.ncu-rep"))):
        name = os.path.basename(rep)[:-len(".ncu-rep")]
        ks = raw(rep)
        summary[name] = ks
        if name in TRAFFIC and ks:
            tb = bytes_of(ks[0])
            if tb:
                traffic[TRAFFIC[name]] = int(tb)
    with open(os.path.join(OUT, "r02_ncu_full.json"), "w") as f:
        json.dump({"note": "ncu --set full --clock-control none, one launch per capture (tools/r02_profile.sh); "
                           "N=256 bf16 ResNet-50 layers, cfg2 = BASELINE configs[1] fp32-accurate",
                   "captures": summary}, f, indent=1)
    with open(os.path.join(OUT, "r02_ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    for nm, note in (("r02_launches_stack", "one ResNet-50 stack training step (global batch 256, eager), all kernels"),
                     ("r02_launches_cfg2", "one cfg2 step (N=32 1x1 256->64 @56, fp32-accurate F + B + U)")):
        p = os.path.join(src, nm + ".csv")
        if os.path.exists(p):
            launches(p, os.path.join(OUT, nm + ".csv"), note)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out"))
