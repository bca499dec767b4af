"""Build an A/B variant of libwmpc.so with extra -D macros: build_variant.py OUT.so -DX=1 ...
(the variant is loaded through WMPC_LIB_EXPERIMENT by the tools, never by the product path)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_10548_b200.build import NVCC_FLAGS, ROOT, SRC

out, defs = sys.argv[1], sys.argv[2:]
cmd = ["nvcc", *NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), "-o", out, *SRC, "-ldl"]
r = subprocess.run(cmd, capture_output=True, text=True)
open(out + ".ptxas.txt", "w").write(r.stderr)
if r.returncode:
    print(r.stderr[-3000:]); sys.exit(1)
print("built", out)
