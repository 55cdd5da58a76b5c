"""Build variant libraries (compile-time switches) for back-to-back A/B timing on one box.
  python tools/ab_variants.py build          # -> paper_2602_05765_b200/variants/*.so
  python tools/ab_variants.py run [mode]     # on the GPU box: time every variant (interleaved)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "paper_2602_05765_b200", "variants")
VARIANTS = {
    "base": (),
}
# name -> git revision whose csrc/ + include/ are built as one more variant
# (the ABI only grew at the end of its structs, so today's binding drives older libraries)
REVISIONS = {"prev": os.environ.get("AB_PREV", "HEAD")} if os.environ.get("AB_PREV", "HEAD") != "none" else {}  # the last commit as a variant


def build_revision(name, rev):
    """Compile `rev`'s csrc with its own include/ into variants/<name>.so (scratch under build/)."""
    from paper_2602_05765_b200 import build as B
    src = os.path.join(B.BUILD, "rev_" + name)
    for sub in ("paper_2602_05765_b200/csrc", "include"):
        os.makedirs(os.path.join(src, sub), exist_ok=True)
        files = subprocess.run(["git", "-C", ROOT, "ls-tree", "--name-only", f"{rev}:{sub}"],
                               capture_output=True, text=True, check=True).stdout.split()
        for f in files:
            blob = subprocess.run(["git", "-C", ROOT, "show", f"{rev}:{sub}/{f}"],
                                  capture_output=True, check=True).stdout
            with open(os.path.join(src, sub, f), "wb") as fh:
                fh.write(blob)
    flags = [f if f != os.path.join(ROOT, "include") else os.path.join(src, "include")
             for f in B._flags()]
    objs = []
    for cu in sorted(os.listdir(os.path.join(src, "paper_2602_05765_b200/csrc"))):
        if not cu.endswith(".cu"):
            continue
        obj = os.path.join(src, cu + ".o")
        subprocess.run([B.NVCC, "-c", os.path.join(src, "paper_2602_05765_b200/csrc", cu), "-o", obj]
                       + flags, check=True, capture_output=True)
        objs.append(obj)
    nd = B.nccl_dir()
    out = os.path.join(VAR, f"{name}.so")
    subprocess.run([B.NVCC, "-shared", "-o", out] + objs + B.ARCH +
                   ["-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
                    "-Xlinker", "-rpath", "-Xlinker", os.path.join(nd, "lib")], check=True)
    print(out)


def build():
    from paper_2602_05765_b200 import build as B
    os.makedirs(VAR, exist_ok=True)
    for name, defs in VARIANTS.items():
        print(B.build(out=os.path.join(VAR, f"{name}.so"), defines=defs))
    for name, rev in REVISIONS.items():
        build_revision(name, rev)


def run(mode="fused", rounds=3):
    """mode: fused | fwd | bwd (tools/prof_fused.py), batcher, scatter or flow (tools/prof_*.py)."""
    res = {}
    for _ in range(rounds):
        for name in list(VARIANTS) + list(REVISIONS):
            if not os.path.exists(os.path.join(VAR, f"{name}.so")):
                continue
            env = dict(os.environ, RLVLA_LIB=os.path.join(VAR, f"{name}.so"))
            if mode == "batcher":
                cmd = [sys.executable, os.path.join(ROOT, "tools", "prof_batcher.py"), "--iters", "30"]
            elif mode == "scatter":
                cmd = [sys.executable, os.path.join(ROOT, "tools", "prof_scatter.py")]
            elif mode == "bench":  # the whole bench step (pipelined), at the box's sustained clocks
                cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", "--no-e2e",
                       "--steps", "40"]
            elif mode == "flow":
                cmd = [sys.executable, os.path.join(ROOT, "tools", "prof_flow.py"), "--rows", "196608"]
                cmd += os.environ.get("FLOW_ARGS", "").split()  # e.g. "--learned --f32"
            elif mode.endswith("32"):  # fp32 logits (the row kernel): fused32 / fwd32 / bwd32
                cmd = [sys.executable, os.path.join(ROOT, "tools", "prof_fused.py"), "--mode", mode[:-2],
                       "--iters", "12", "--f32", "--rows", "32768"]
            else:
                cmd = [sys.executable, os.path.join(ROOT, "tools", "prof_fused.py"), "--mode", mode,
                       "--iters", "12"]
            out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
            lines = out.stdout.strip().splitlines()
            if out.returncode != 0 or not lines:
                res.setdefault(name, []).append("failed")
                continue
            d = json.loads(lines[-1])
            if mode == "batcher":
                res.setdefault(name, []).append((round(d["poll_us_min"], 2), round(d["poll_us_median"], 2)))
            elif mode == "flow":
                res.setdefault(name, []).append((round(d["us_min"], 1), round(d["us_median"], 1)))
            elif mode == "scatter":
                res.setdefault(name, []).append(round(d["us_per_call"], 2))
            elif mode == "bench":
                res.setdefault(name, []).append((round(d["ms_per_step"], 3), round(d["roofline"]["kernel_ms"], 3),
                                                 (d.get("clocks") or {}).get("sm_mhz")))
            else:
                res.setdefault(name, []).append((round(d["ms_min"], 3), round(d["ms_avg"], 3)))
    print(json.dumps(res))


if __name__ == "__main__":
    {"build": build, "run": lambda: run(*(sys.argv[2:3] or ["fused"]))}[sys.argv[1]]()
