"""Build libdlrmb200.so with extra nvcc defines into gpurun_var/<name>/ (A/B
experiments; load it with DLRM_B200_LIB=<path>).

    python scripts/build_variant.py chunk2 -DDLRM_GEMM_CHUNK=2
"""
import glob, os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1906_00091_b200.build import ARCH, CSRC, FLAGS, NVCC  # noqa: E402

name = sys.argv[1]
defs = [a for a in sys.argv[2:] if not a.startswith("--src=")]
# --src=<file.cu>=<path>: compile <path> in place of csrc/<file.cu>
over = dict(a[6:].split("=", 1) for a in sys.argv[2:] if a.startswith("--src="))
out = os.path.join(ROOT, "gpurun_var", name)
os.makedirs(out, exist_ok=True)
srcs = [over.get(os.path.basename(x), x) for x in sorted(glob.glob(os.path.join(CSRC, "*.cu")))]
objs = [os.path.join(out, os.path.basename(s)[:-3] + ".o") for s in srcs]

def cc(a):
    s, o = a
    subprocess.run([NVCC, *FLAGS, f"-I{CSRC}", *defs, "-c", s, "-o", o], check=True,
                   capture_output=True)

with ThreadPoolExecutor(8) as ex:
    list(ex.map(cc, zip(srcs, objs)))
subprocess.run([NVCC, *ARCH, "-shared", "-o", os.path.join(out, "libdlrmb200.so"), *objs], check=True)
print(os.path.join(out, "libdlrmb200.so"))
