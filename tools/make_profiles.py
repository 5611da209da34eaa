"""Dev tool: summarise gpurun_out ncu captures into the committed profiles/.

usage: python tools/make_profiles.py <launches.csv> <full.ncu-rep> <bench.json> [<stack_bench.json>]"""
import csv
import json
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr, ks = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                ks.append((d["Kernel Name"], float(d["Metric Value"].replace(",", ""))))
    first = min(i for i, k in enumerate(ks) if "spin_kernel" in k[0])
    step = []
    for n, t in ks[first + 1:]:
        if "spin_kernel" in n or "FillFunctor" in n or "reduce_kernel_impl" in n or "at::native" in n:
            break
        step.append((n, t))
    tot = sum(t for _, t in step)
    with open(out, "w") as f:
        f.write("# r01 launch list: one bench.py step (cfg2 fp32-accurate F+B+U), "
                "ncu --metrics gpu__time_duration.sum --clock-control none (ns)\n")
        f.write("# serialised and cold-cache under ncu: compare SHARES with the bench's live CUDA-event kernel times\n")
        f.write("kernel,ns,share\n")
        for n, t in step:
            f.write(f"{n.split('(')[0].replace('void ', '')},{int(t)},{t / tot:.3f}\n")


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(raw.splitlines())
    h = next(r)
    u = dict(zip(h, next(r)))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
            "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__issue_active.avg.pct_of_peak_sustained_elapsed"]
    ks = []
    roles = ["fwd (conv_fwd_kernel<1,3,1>: A pieces in TMEM)", "bwd (same kernel on the dual problem)",
             "upd (conv_upd_ts_kernel<3,1>: activations in TMEM)"]
    for v, role in zip(r, roles):
        d = dict(zip(h, v))
        e = {"Kernel Name": d["Kernel Name"].split("(")[0], "pass": role}
        for k in keys:
            e[k] = (d.get(k, "") + " " + u.get(k, "")).strip()
        ks.append(e)
    json.dump({"note": "r01 ncu --set full --clock-control none, one launch each of the cfg2 F/B/U conv kernels "
                       "(bench.py --steps 1 --warmup 0); dram bytes per launch feed roofline.traffic",
               "kernels": ks}, open(out, "w"), indent=1)
    for e in ks:
        print(e["pass"][:4], e["gpu__time_duration.sum"], e["dram__bytes_read.sum"], e["dram__bytes_write.sum"])


if __name__ == "__main__":
    launches(sys.argv[1], "profiles/r01_launches_cfg2.csv")
    full(sys.argv[2], "profiles/r01_ncu_full_cfg2.json")
    for src, dst in zip(sys.argv[3:], ["profiles/r01_bench_cfg2.json", "profiles/r01_bench_resnet50.json"]):
        line = [ln for ln in open(src) if ln.startswith("{")][-1]
        open(dst, "w").write(line)
