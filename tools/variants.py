"""Build library variants with extra -D defines and time each with kbench.

    python tools/variants.py build NAME=DEF1,DEF2 ...   (here, nvcc cross-compiles)
    python tools/variants.py run NAME ...               (GPU box: kbench per variant)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIBDIR = os.path.join(ROOT, "paper_2603_00145_b200", "_lib")


def main():
    mode, specs = sys.argv[1], sys.argv[2:]
    extra = []
    if "--" in specs:  # run: arguments after -- go to kbench
        extra = specs[specs.index("--") + 1:]
        specs = specs[:specs.index("--")]
    if mode == "build":
        from paper_2603_00145_b200 import _build
        for sp in specs:
            name, _, defs = sp.partition("=")
            out = os.path.join(LIBDIR, f"var_{name}.so")
            _build.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
            print("built", out)
    else:
        for name in specs:
            env = dict(os.environ, MGAUSS_B200_LIB=os.path.join(LIBDIR, f"var_{name}.so"))
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "kbench.py"), *extra], env=env,
                               capture_output=True, text=True)
            print("==", name, (r.stdout.strip().splitlines() or [r.stderr[-400:]])[-1], flush=True)


if __name__ == "__main__":
    main()
