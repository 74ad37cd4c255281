"""configs[4] (M5): Qwen3-8B sparsity sweep 0.1/1/10/50 % x {uniform, rowblock}, plus
M1/M2 and the fp32 variant — one bench.py line per point, run sequentially on one GPU.
Usage (GPU box): python scripts/sweep.py > gpurun_out/sweep.jsonl"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
POINTS = [("M1", None, None), ("M2", None, None)]
POINTS += [("M5", rho, pat) for pat in ("uniform", "rowblock") for rho in (0.001, 0.01, 0.1, 0.5)]


def main():
    extra = sys.argv[1:]
    for cfg, rho, pat in POINTS:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "10", "--warmup", "3",
               "--no-e2e", "--no-cpu-baseline"] + extra
        if rho is not None:
            cmd += ["--rho", str(rho), "--pattern", pat]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 and r.stdout.strip() else None
        if line is None:
            print(json.dumps({"config": cfg, "rho": rho, "pattern": pat, "error": r.stderr[-2000:]}), flush=True)
            continue
        d = json.loads(line)
        print(json.dumps({"config": cfg, "rho": d["config"]["rho"], "pattern": d["config"]["pattern"],
                          "value_GBps": d["value"], "ms_per_step": d["ms_per_step"],
                          "payload_ratio": d["payload"]["ratio"], "body_bytes": d["payload"]["body_bytes"],
                          "index_bytes_per_entry": d["payload"]["index_bytes_per_entry"],
                          "k1_GBps": d["roofline"]["achieved"], "kernel_ms": d["kernel_ms_per_step"]}),
              flush=True)


if __name__ == "__main__":
    main()
