"""Symmetric (LDLT) against unsymmetric (PLDUQ) elimination of the same matrices on the
device -- the comparison of the paper's timing table, which f-4
(the standalone ffb_plduq) exists for.

    python tools/pluq_vs_ldlt.py [n ...]          # default 2048 4096 8192

Families: config 1 (dense symmetric, generic rank profile) and config 5 (rank n/2,
random rank profile matrix) at each n.  Both times are device times of the
factorization alone: LDLT = ffb_ldlt_device bracketed by CUDA events, PLDUQ = the
engine's own per-call timer (FFB_PLDUQ_TRACE: the PLDUQ of the uploaded matrix between
two stream synchronisations, without the host transfers).  The PLDUQ phase runs in a
child process because that trace synchronises every PLDUQ and would slow the LDLT runs.
One JSON line per (family, n).
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def sizes(argv):
    return [int(a) for a in argv if a.isdigit()] or [2048, 4096, 8192]


def phase_pluq(ns):
    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200 import configs

    path = os.environ["FFB_PLDUQ_TRACE"]
    for c in (1, 5):
        for n in ns:
            w = configs.CONFIGS[c].scaled(n)
            a = configs.generate(w)
            best, rank = None, None
            for _ in range(2):
                open(path, "w").close()
                f = ffb.plduq(a, w.p)
                rows = [ln.split() for ln in open(path).read().splitlines() if ln.strip()]
                ms = float(rows[-1][3])
                best = ms if best is None else min(best, ms)
                rank = f.rank
            print(json.dumps(dict(config=c, n=n, pluq_ms=best, rank=rank)), flush=True)


def phase_ldlt(ns):
    import torch

    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200 import configs
    from paper_1802_10453_b200.device import DeviceBuffers, ldlt_device

    ctx = ffb.default_context(0)
    res = {}
    for c in (1, 5):
        for n in ns:
            w = configs.CONFIGS[c].scaled(n)
            a0 = configs.generate_device(w, ctx)
            a = torch.empty_like(a0)
            out = DeviceBuffers(n)
            ts = []
            for it in range(4):
                a.copy_(a0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rank = ldlt_device(a, w.p, ffb.SytrfConfig(), ctx, out)
                e1.record()
                torch.cuda.synchronize()
                if it:
                    ts.append(e0.elapsed_time(e1))
            res[(c, n)] = (sorted(ts)[len(ts) // 2], int(rank.rank))
    return res


def main():
    ns = sizes(sys.argv[1:])
    if "--phase-pluq" in sys.argv:
        phase_pluq(ns)
        return
    ld = phase_ldlt(ns)
    with tempfile.NamedTemporaryFile(suffix=".txt") as tf:
        env = dict(os.environ, FFB_PLDUQ_TRACE=tf.name)
        cp = subprocess.run([sys.executable, os.path.abspath(__file__), "--phase-pluq"] + [str(n) for n in ns],
                            env=env, capture_output=True, text=True)
        if cp.returncode:
            sys.stderr.write(cp.stderr)
            sys.exit(cp.returncode)
        outp = cp.stdout
    for ln in outp.splitlines():
        d = json.loads(ln)
        ms, rank = ld[(d["config"], d["n"])]
        d.update(ldlt_ms=round(ms, 3), ldlt_rank=rank, pluq_ms=round(d["pluq_ms"], 3),
                 pluq_over_ldlt=round(d["pluq_ms"] / ms, 2),
                 family="generic rank profile (config 1)" if d["config"] == 1 else
                 "rank n/2, random rank profile matrix (config 5)")
        print(json.dumps(d))


if __name__ == "__main__":
    main()
