"""Step-time ablation at a bench config (measurement only: the listed
stages are left out of the captured step, so results are wrong): how much of
the device step time each stage holds on the critical path.
    python scripts/ablate.py [config]"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
cases = sys.argv[2].split(";") if len(sys.argv) > 2 else [
    "", "apply", "lookup", "ia_fwd", "ia_bwd", "ia_fwd,ia_bwd", "bot", "top", "apply,lookup",
    "top,bot", "apply_early"]
for c in cases:
    env = dict(os.environ, DLRM_ABLATE=c)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "30",
                        "--warmup", "5", "--quick"], env=env, capture_output=True,
                       text=True, cwd=ROOT)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    ms = json.loads(line[-1])["ms_per_step"] if line else None
    print(f"{c or 'none':22s} {ms}", flush=True)
