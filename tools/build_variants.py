"""Build experimental libpbit variants (extra -D flags) into build/var/ in parallel:
python tools/build_variants.py name=-DX=1,-DY=2 ..."""
import importlib.util
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_cs_0511020_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
os.makedirs(os.path.join(ROOT, "build", "var"), exist_ok=True)
procs = []
for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    out = os.path.join(ROOT, "build", "var", f"libpbit_{name}.so")
    procs.append((name, subprocess.Popen(b.nvcc_cmd(out, extra=[f for f in flags.split(",") if f]))))
bad = [name for name, p in procs if p.wait() != 0]
print("built", [n for n, _ in procs if n not in bad], "failed", bad)
