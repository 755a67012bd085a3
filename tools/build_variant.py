"""Build an ablation variant of libfedb200.so: `python tools/build_variant.py NAME -DFLAG ...`
recompiles every csrc/*.cu with the extra flags into tools/libfedb200_NAME.so (load it with
FB_LIB_PATH). Used for A/B experiments only; the product library is built by build.py."""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_10853_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.CSRC, "build", "v_" + name)
os.makedirs(out_dir, exist_ok=True)


# SRC_OVERRIDE="gemm_sm100.cu=/path/to/other.cu,..." swaps individual sources (A/B against an old revision)
OVR = dict(x.split("=", 1) for x in os.environ.get("SRC_OVERRIDE", "").split(",") if x)


def comp(src):
    obj = os.path.join(out_dir, os.path.basename(src).replace(".cu", ".o"))
    src = OVR.get(os.path.basename(src), src)
    r = subprocess.run([B.NVCC, *B.FLAGS, "-I", B.CSRC, *flags, "-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return obj


with cf.ThreadPoolExecutor(os.cpu_count() or 4) as ex:
    objs = list(ex.map(comp, sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))))
out = os.path.join(ROOT, "tools", f"libfedb200_{name}.so")
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs,
                "-Xcompiler", "-fPIC"], check=True)
print(out)
