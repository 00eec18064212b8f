"""Time the UNMODIFIED reference (oracle/_ref) single-threaded on each BASELINE.json
configuration, on the host it runs on (run it on a GPU box: the CPU baseline is quoted for
the box's host cores).  Each configuration is measured at the largest size of its family
whose predicted time fits the cap (default 600 s); when that is smaller than
the stated size the full-size time is an n^3 extrapolation, labelled as such.

    python tools/cpu_reference_configs.py [--cap 600] [--out gpurun_out/cpu_reference_configs.json]

Each timed call runs in its own process under a hard timeout of the cap.  Inputs come from
oracle/gen_oracle.c (the product library is not loaded).
"""
import argparse
import json
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {  # (n, p, rank parameter, seed) -- paper_1802_10453_b200/configs.py
    1: (1024, 131, 0, 1), 2: (4096, 131, 2048, 2), 3: (8192, 8388593, 0, 3),
    4: (16384, 131, 0, 4), 5: (32768, 131, 16384, 5),
}


def _one(c, n, q):
    from oracle.bind import Checker
    N, p, R, seed = CONFIGS[c]
    r = (R * n) // N if R else 0
    a = Checker("oracle").generate(c, n, r, p, seed)
    ref = Checker("ref")
    t0 = time.perf_counter()
    f = ref.ldlt(p, a, "cascade", 64)
    q.put((time.perf_counter() - t0, f.rank))


def timed(c, n, cap):
    q = mp.Queue()
    pr = mp.Process(target=_one, args=(c, n, q))
    pr.start()
    pr.join(cap + 120)  # + input generation
    if pr.is_alive():
        pr.kill()
        pr.join()
        return None
    return q.get() if not q.empty() else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cap", type=float, default=600.0)
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cpu_reference_configs.json"))
    args = ap.parse_args()
    res = {"how": "unmodified reference (oracle/_ref, g++ -O2) single-threaded ffldl::ldlt, "
                  "Cascade T=64; wall time of the call; inputs from oracle/gen_oracle.c",
           "cap_s": args.cap, "host": platform.node(), "cpu": platform.processor(),
           "nproc": os.cpu_count(), "configs": {}}
    for c in (int(x) for x in args.configs.split(",")):
        N = CONFIGS[c][0]
        rows = []
        n = min(N, 1024)
        while True:
            r = timed(c, n, args.cap)
            if r is None:
                break
            rows.append({"n": n, "s": r[0], "rank": r[1]})
            print(c, n, r, flush=True)
            if n >= N:
                break
            pred = r[0] * 8.0
            if pred > args.cap * 0.8:
                break
            n *= 2
        last = rows[-1]
        out = {"n": N, "measured": rows}
        if last["n"] == N:
            out["full_size_s"] = last["s"]
            out["full_size_kind"] = "measured"
        else:
            out["full_size_s"] = last["s"] * (N / last["n"]) ** 3
            out["full_size_kind"] = f"extrapolated n^3 from n={last['n']} (exceeds the {args.cap:.0f} s cap)"
        out["tops"] = 2.0 * N ** 3 / 3.0 / out["full_size_s"] / 1e12
        res["configs"][str(c)] = out
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
