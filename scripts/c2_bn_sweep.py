"""C2 main-path time (EMA predictor) and per-phase worker times for GEMM tile widths (debug)."""
import os, sys, subprocess
for fwd in ("64", "128", "256"):
    for dw in ("64", "128", "256"):
        env = dict(os.environ, LBBSP_BN_FWD=fwd, LBBSP_BN_DW=dw)
        out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "c2_timeline.py")],
                             env=env, capture_output=True, text=True).stdout.strip().splitlines()
        ema = [l for l in out if l.startswith("ema")]
        print(f"fwd={fwd} dw={dw}: " + (ema[-1][:40] + " ... " + ema[-1][ema[-1].index("phases"):] if ema else "fail"))
