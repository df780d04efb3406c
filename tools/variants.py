"""Build library variants (compile-time switches) into tools/_v/<name>.so, in parallel.
    python tools/variants.py name1="-DFOO=1 -DBAR=0" name2="..."
(development aid for kernel A/B experiments; the .so files travel with gpurun)"""
import os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2510_20271_b200 import build as B
procs = []
for arg in sys.argv[1:]:
    name, _, flags = arg.partition("=")
    out = ROOT / "tools" / "_v" / f"{name}.so"
    out.parent.mkdir(exist_ok=True)
    cmd = [os.environ.get("NVCC", "nvcc"), *B.NVCC_FLAGS, *flags.split(), "-o", str(out),
           *[str(B.CSRC / s) for s in B.SOURCES]]
    procs.append((name, subprocess.Popen(cmd, stderr=subprocess.PIPE, text=True)))
for name, p in procs:
    _, err = p.communicate()
    print(name, "ok" if p.returncode == 0 else "FAILED\n" + err[-2000:])
