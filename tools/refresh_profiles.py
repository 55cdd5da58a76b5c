"""Regenerate profiles/<round>/ from one set of gpurun outputs (tag = the prefix the
tools/gpu_*.sh scripts wrote under gpurun_out/):

  python tools/refresh_profiles.py r1 r1y

reads <tag>_bench/_ref/_prof/_launches/_fused (gpu_round + gpu_ncu_*), <tag>_bprof/_bpoll
(gpu_batcher), <tag>_fprof/_flow (gpu_flow), <tag>2_bench / <tag>4_bench (gpu_mgpu) and
writes SUMMARY.md (+ raw CSVs via summarize_profiles.py), BATCHER.md, FLOW.md and the
jsonl files. Existing narrative sections of BATCHER.md / FLOW.md below their tables are kept."""
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def jl(path):
    return [json.loads(l) for l in open(path) if l.startswith("{")]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return out, {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}


def main():
    rnd, tag = sys.argv[1], sys.argv[2]
    prof = os.path.join(ROOT, "profiles", rnd)
    pre = os.path.join(OUT, tag)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_profiles.py"), rnd, pre], check=True)
    shutil.copy(pre + "_ref.jsonl", os.path.join(prof, "bench_reference.jsonl"))
    for n in (2, 4):
        src = os.path.join(OUT, f"{tag}{n}_bench.log")
        if os.path.exists(src):
            with open(os.path.join(prof, f"bench_n{n}.jsonl"), "w") as f:
                for d in jl(src):
                    f.write(json.dumps(d) + "\n")
            topo = os.path.join(OUT, f"{tag}{n}_topo.txt")
            if os.path.exists(topo):
                shutil.copy(topo, os.path.join(prof, f"topo_{n}gpu.txt"))
    # SUMMARY.md additions: NEXT-2 knob timings (kept file), scaling, stages, reference arm
    s = open(os.path.join(prof, "SUMMARY.md")).read()
    vf = os.path.join(prof, "prof_fused_variants.jsonl")
    if os.path.exists(vf):
        s += ("\n## NEXT-2 loss knobs on the fused call (tools/prof_fused.py --variant, one box, back to back)\n\n"
              "| variant | ms avg | ms min | GB/s best |\n|---|---|---|---|\n")
        for d in jl(vf):
            s += f"| {d['variant']} | {d['ms_avg']:.3f} | {d['ms_min']:.3f} | {d['GBps_best']:.0f} |\n"
        s += ("\n`dual` and `kl` ride in the same epilogue (kl adds 4 B/row of logp_ref); `ent` (entropy-bonus "
              "gradient) runs pass C from x (one more ex2 per element).\n")
    b1 = jl(os.path.join(prof, "bench.jsonl"))[-1]
    rows = [(1, b1)]
    for n in (2, 4):
        p = os.path.join(prof, f"bench_n{n}.jsonl")
        if os.path.exists(p):
            rows.append((n, jl(p)[-1]))
    s += ("\n## Weak scaling (64 envs per GPU, one box; statistics reduced in-kernel over NVLink)\n\n"
          "| GPUs | env-steps/s | ms/step | per-GPU fused frac | e2e env-steps/s | sm MHz |\n|---|---|---|---|---|---|\n")
    for n, b in rows:
        s += (f"| {n} | {b['value'] / 1e6:.2f} M | {b['ms_per_step']:.3f} | {b['roofline']['frac']:.3f} | "
              f"{b['e2e']['value'] / 1e6:.2f} M | {b['clocks']['sm_mhz']} |\n")
    s += "\nThe driver computes its own scaling efficiency from these values.\n"
    s += f"\nStages at N=1 (CUDA event nodes inside the timed graph): `{json.dumps(b1['stages'])}`\n"
    ref = jl(os.path.join(prof, "bench_reference.jsonl"))[-1]
    s += (f"\nReference arm (`bench.py --impl reference`, the CPU oracle on the box's host): {ref['value']:.1f} "
          f"{ref['unit']} ({ref['cpu_baseline']['sample']}; {ref['cpu_baseline'].get('host', '')}).\n")
    open(os.path.join(prof, "SUMMARY.md"), "w").write(s)
    # BATCHER.md table rows
    if os.path.exists(pre + "_bprof.log"):
        shutil.copy(pre + "_bprof.log", os.path.join(prof, "prof_batcher.jsonl"))
        bp = jl(pre + "_bprof.log")[-1]
        out, m = raw(pre + "_bpoll.ncu-rep")
        open(os.path.join(prof, "ncu_full_batch_poll_raw.csv"), "w").write(out)
        b = open(os.path.join(prof, "BATCHER.md")).read()
        vals = {
            "poll (fires, gathers 64), CUDA events, median / min": f"{bp['poll_us_median']:.1f} / {bp['poll_us_min']:.1f} us",
            "achieved (alg. bytes / median)": f"{bp['GBps_median']:.0f} GB/s = {bp['GBps_median'] / 6548.8 * 100:.0f} % of 6548.8 GB/s",
            "idle poll (no trigger), median": f"{bp['idle_poll_us_median']:.1f} us",
            "offer of 64 requests (zero-copy), median": f"{bp['offer_us_median']:.1f} us",
            "steady tick loop (offer + firing poll, PDL), per tick": f"{bp['tick_loop']['us_per_tick']:.1f} us ({bp['tick_loop']['GBps']:.0f} GB/s)",
            "torch.index_select of the same rows (no queue logic), median": f"{bp['torch_index_select_us_median']:.1f} us",
            "ncu: poll duration (cold, serialised)": f"{float(m['gpu__time_duration.sum'][1]):.2f} {m['gpu__time_duration.sum'][0]}",
        }
        for k, v in vals.items():
            b = re.sub(r"\| " + re.escape(k) + r" \| [^\n]*\|", f"| {k} | {v} |", b)
        st = bp.get("staged_tick_loop", {})
        if st:
            b = re.sub(r"\| env slots \(copy into slots at offer, gather at poll\) \| [^\n]*\|",
                       f"| env slots (copy into slots at offer, gather at poll) | {st['env_slots']['bytes_per_tick'] / 1e6:.1f} MB | "
                       f"{st['env_slots']['us_per_tick']:.1f} | {st['env_slots']['GBps']:.0f} |", b)
            b = re.sub(r"\| FIFO rows \(copy into FIFO rows at offer, batch read in place\) \| [^\n]*\|",
                       f"| FIFO rows (copy into FIFO rows at offer, batch read in place) | {st['fifo_rows']['bytes_per_tick'] / 1e6:.1f} MB | "
                       f"{st['fifo_rows']['us_per_tick']:.1f} | {st['fifo_rows']['GBps']:.0f} |", b)
        open(os.path.join(prof, "BATCHER.md"), "w").write(b)
    # FLOW.md table
    if os.path.exists(pre + "_fprof.log"):
        shutil.copy(pre + "_fprof.log", os.path.join(prof, "prof_flow.jsonl"))
        out, m = raw(pre + "_flow.ncu-rep")
        open(os.path.join(prof, "ncu_full_flow_tma_raw.csv"), "w").write(out)
        f = open(os.path.join(prof, "FLOW.md")).read()
        tab = ["| rows | K x D | mu | ln sigma | alg. bytes | median us | GB/s | % of 6548.8 |", "|---|---|---|---|---|---|---|---|"]
        for d in jl(pre + "_fprof.log"):
            tab.append(f"| {d['rows']} | {d['K']} x {d['D']} | {d['mu_dtype']} | {'learned' if d['learned_log_std'] else 'schedule'} | "
                       f"{d['alg_bytes'] / 1e6:.1f} MB | {d['us_median']:.1f} | {d['GBps_median']:.0f} | {d['GBps_median'] / 6548.8 * 100:.0f} % |")
        f = re.sub(r"\| rows \| K x D \|.*?\n\n", "\n".join(tab) + "\n\n", f, flags=re.S)
        g = lambda k: m[k][1]  # noqa: E731
        f = re.sub(r"ncu \(196,608 rows, bf16 mu, schedule\):\n\n.*?\n\n",
                   "ncu (196,608 rows, bf16 mu, schedule):\n\n"
                   f"- duration {float(g('gpu__time_duration.sum')):.1f} us; DRAM read {g('dram__bytes_read.sum')} {m['dram__bytes_read.sum'][0]}, "
                   f"write {g('dram__bytes_write.sum')} {m['dram__bytes_write.sum'][0]} (algorithmic: 335 MB read, 110 MB written)\n"
                   f"- issue active {float(g('smsp__issue_active.avg.pct_of_peak_sustained_active')):.1f} %, warps active "
                   f"{float(g('sm__warps_active.avg.pct_of_peak_sustained_active')):.1f} %, registers {g('launch__registers_per_thread')}\n"
                   f"- instructions per decision step {float(g('smsp__inst_executed.sum')) / 196608:.0f} (warp level)\n\n", f, flags=re.S)
        open(os.path.join(prof, "FLOW.md"), "w").write(f)
    print("refreshed", prof)


if __name__ == "__main__":
    main()
