"""Summarise a round's ncu evidence into profiles/<round>/:
  python tools/summarize_profiles.py <round> <gpurun_out prefix>
reads <prefix>_fused.ncu-rep (ncu --set full, one fused launch), <prefix>_launches.csv
(gpu__time_duration.sum launch list of `bench.py --steps 2 --warmup 1`), <prefix>_bench.log
and <prefix>_prof.log; writes raw CSVs, traffic_fused.json and SUMMARY.md."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return out, {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"msecond": 1e3, "ms": 1e3, "usecond": 1.0, "us": 1.0, "nsecond": 1e-3, "ns": 1e-3}[d["Metric Unit"]]
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    return agg


def main():
    rnd, pre = sys.argv[1], sys.argv[2]
    outdir = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(outdir, exist_ok=True)
    raw_csv, m = ncu_raw(pre + "_fused.ncu-rep")
    open(os.path.join(outdir, "ncu_full_fused_raw.csv"), "w").write(raw_csv)
    shutil.copy(pre + "_launches.csv", os.path.join(outdir, "launches_bench_steps2.csv"))
    bench = [json.loads(l) for l in open(pre + "_bench.log") if l.startswith("{")]
    prof = [json.loads(l) for l in open(pre + "_prof.log") if l.startswith("{")]
    with open(os.path.join(outdir, "bench.jsonl"), "w") as f:
        for b in bench:
            f.write(json.dumps(b) + "\n")
    with open(os.path.join(outdir, "prof_fused_modes.jsonl"), "w") as f:
        for p in prof:
            f.write(json.dumps(p) + "\n")
    g = lambda k: float(m[k][1]) if k in m else float("nan")  # noqa: E731
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    unit = m["dram__bytes_read.sum"][0]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "byte": 1.0}[unit]
    rd, wr = rd * scale, wr * scale
    dur_ms = g("gpu__time_duration.sum") * ({"ms": 1.0, "us": 1e-3}[m["gpu__time_duration.sum"][0]])
    alg = 229376 * (2 * 32000 * 2 + 12) + 4096 * 16
    json.dump({"kernel": "lp_tma_kernel<1> (fused log-softmax + PPO fwd/bwd), 229376 x 32000 bf16",
               "source": f"profiles/{rnd}/ncu_full_fused_raw.csv (ncu --set full, one launch)",
               "dram_bytes_read": rd, "dram_bytes_write": wr, "bytes_per_launch": rd + wr,
               "alg_bytes_per_launch": alg, "ncu_duration_ms": dur_ms, "rows_per_launch": 229376,
               "vocab": 32000}, open(os.path.join(ROOT, "profiles", "traffic_fused.json"), "w"),
              indent=1)
    stalls = sorted(((float(v[1]), k.replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", "")) for k, v in m.items()
                     if k.startswith("smsp__average_warps_issue_stalled_")
                     and k.endswith("per_issue_active.ratio") and v[1]), reverse=True)[:6]
    agg = launch_table(pre + "_launches.csv")
    tot = sum(v for _, v in agg.values())
    b = bench[-1] if bench else {}
    lines = [f"# Profile summary — {rnd}", "",
             "Commands (one GPU, B200, under `gpurun`): `python bench.py` (the bench line);",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over",
             "`python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline` (launch list);",
             "`ncu --set full --clock-control none --import-source on -k regex:lp_tma_kernel -s 1 -c 1`",
             "over `python tools/prof_fused.py --mode fused --iters 1` (dominant kernel).", "",
             "## Dominant kernel: fused log-softmax + PPO (`lp_tma_kernel<FUSED>`)", "",
             "| quantity | value |", "|---|---|",
             f"| ncu duration (cold, serialised) | {dur_ms:.3f} ms |",
             f"| DRAM read / write per launch | {rd / 1e9:.3f} / {wr / 1e9:.3f} GB |",
             f"| traffic / algorithmic bytes | {(rd + wr) / alg:.4f} |",
             f"| DRAM throughput (ncu, % of theoretical) | {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} % |",
             f"| achieved (traffic / ncu duration) | {(rd + wr) / dur_ms / 1e6:.0f} GB/s |",
             f"| XU (MUFU) pipe, % of peak active | {g('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):.1f} % |",
             f"| issue active | {g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} % |",
             f"| warp instructions per row | {g('smsp__inst_executed.sum') / 229376:.0f} |",
             f"| registers / thread, local-memory instructions | {g('launch__registers_per_thread'):.0f}, {g('sass__inst_executed_local_loads') + g('sass__inst_executed_local_stores'):.0f} |",
             "", "Top stall reasons (warps per issue): " + ", ".join(f"{k} {v:.2f}" for v, k in stalls), ""]
    if prof:
        lines += ["## CUDA-event timing of the three modes (tools/prof_fused.py, 229,376 x 32000 bf16)", "",
                  "| mode | ms avg | ms min | GB/s avg | GB/s best |", "|---|---|---|---|---|"]
        for p in prof:
            lines.append(f"| {p['mode']} | {p['ms_avg']:.3f} | {p['ms_min']:.3f} | {p['GBps_avg']:.0f} | {p['GBps_best']:.0f} |")
        lines.append("")
    lines += ["## Launch list of `bench.py --steps 2 --warmup 1` (ncu, serialised, cold cache)", "",
              "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
        lines.append(f"| `{k[:70]}` | {n} | {v:.1f} | {v / n:.2f} | {100 * v / tot:.1f} % |")
    if b:
        r = b["roofline"]
        lines += ["", "## Bench line (same round)", "",
                  f"value {b['value']:.4g} {b['unit']}, {b['ms_per_step']:.3f} ms/step, fused kernel "
                  f"{r['kernel_ms']:.3f} ms = {r['achieved']:.0f} GB/s = {100 * r['frac']:.1f} % of "
                  f"{r['peak']} GB/s ({r['peak_source']}); kernel share of step "
                  f"{100 * r['kernel_share_of_step']:.1f} %; clocks {b.get('clocks')}."]
    open(os.path.join(outdir, "SUMMARY.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
