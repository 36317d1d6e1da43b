"""Build an A/B variant of libpe.so with extra -D flags (experiments only;
load it with PE_LIB_OVERRIDE=<path>).  Usage:
python scripts/build_variant.py <out.so> -DPE_LONG_STAGES=5 ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_16932_b200 import build as b  # noqa: E402

out = sys.argv[1]
cmd = ["nvcc", *b.NVCC_FLAGS, *sys.argv[2:], "-I", os.path.join(ROOT, "include"), "-I", b.CSRC,
       *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-ldl", "-o", out]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stderr[-4000:])
    sys.exit(1)
print(out, "ok")
