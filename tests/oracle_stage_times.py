"""The oracle timed per stage on the host (configs 1 and 2 "oracle per stage",
config 5 "Vincent's algorithm on 1 core").  A helper script of the test infrastructure (the
oracle may only be run from tests/, smoke() and bench.py's CPU legs); single-threaded.
usage: python tests/oracle_stage_times.py [out.json]"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import make_stress  # noqa: E402
from synth.hne import make_config_tile  # noqa: E402

STAGES = ["S1 CD", "S2 RBC", "S3 open", "S4 recon", "S5 area", "S6 fill", "S7 EDT", "S8 markers",
          "S9 watershed", "S10 bwlabel", "S11 features"]


def main():
    out = {"host_cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")
           if os.path.exists("/proc/cpuinfo") else None, "threads": 1, "configs": []}
    for cfg, reps in ((1, 3), (2, 1)):
        rgb = make_config_tile(cfg)
        runs = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = oracle.process_tile(rgb, with_times=True)
            runs.append((time.perf_counter() - t0, r[-1]))
        whole = statistics.median(x[0] for x in runs)
        per = [statistics.median(x[1][i] for x in runs) for i in range(11)]
        out["configs"].append({"config": cfg, "reps": reps, "s_whole": whole,
                               "s_per_stage": {STAGES[i]: round(per[i], 4) for i in range(11)}})
        print(json.dumps(out["configs"][-1]), flush=True)
    cases = []
    for kind in ("serpentine", "spiral"):
        for ramp in (False, True):
            marker, mask, _ = make_stress(kind, 4096, ramp)
            t0 = time.perf_counter()
            rec = oracle.recon_u8(marker, mask)
            dt = time.perf_counter() - t0
            cases.append({"case": f"{kind} {'ramp' if ramp else 'binary'}", "s": round(dt, 3),
                          "recon_eq_mask": bool((rec == mask).all())})
    out["configs"].append({"config": 5, "oracle": "Vincent's hybrid reconstruction, 1 core (or_recon_u8)",
                           "cases": cases})
    print(json.dumps(out["configs"][-1]), flush=True)
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
