"""Config-size parity with the reference (BASELINE.json configs[0]-[4]) ->
profiles/parity_<tag>.json with every comparison's agreement counts.

  python tools/parity_configs.py [--configs 1,2,3,4,5] [--tag r2]

Runs on the GPU box (the checkers use every host core); the records and the
assertions are the ones tests/test_gpu_configs.py makes."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--tag", default="r2")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import config_parity as cp
    env = cp.Env()
    path = args.out or os.path.join(ROOT, "profiles", f"parity_{args.tag}.json")
    res = {"threads": env.threads, "seed": cp.SEED, "configs": {}}
    if os.path.exists(path):
        try:
            res = json.load(open(path))
        except Exception:
            pass
    import platform
    res["host"] = {"cpu": platform.processor() or platform.machine(), "threads": env.threads}
    for c in [int(v) for v in args.configs.split(",") if v]:
        t0 = time.perf_counter()
        rec = cp.RUNNERS[c](env)
        rec["wall_s"] = time.perf_counter() - t0
        rec["all_ok"] = cp.all_ok(rec)
        res["configs"][str(c)] = rec
        print(f"config {c}: all_ok={rec['all_ok']} ({rec['wall_s']:.1f} s)", flush=True)
        with open(path, "w") as f:
            json.dump(res, f, indent=1, default=float)
    print(path)


if __name__ == "__main__":
    main()
