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
    "element_clamp": ("RLVLA_PACKED_CLAMP=0",),
}


def build():
    from paper_2602_05765_b200 import build as B
    os.makedirs(VAR, exist_ok=True)
    for name, defs in VARIANTS.items():
        print(B.build(out=os.path.join(VAR, f"{name}.so"), defines=defs))


def run(mode="fused", rounds=3):
    res = {}
    for _ in range(rounds):
        for name in VARIANTS:
            env = dict(os.environ, RLVLA_LIB=os.path.join(VAR, f"{name}.so"))
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "prof_fused.py"),
                                  "--mode", mode, "--iters", "12"], env=env, capture_output=True,
                                 text=True, timeout=300)
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res.setdefault(name, []).append((round(d["ms_min"], 3), round(d["ms_avg"], 3)))
    print(json.dumps(res))


if __name__ == "__main__":
    {"build": build, "run": lambda: run(*(sys.argv[2:3] or ["fused"]))}[sys.argv[1]]()
