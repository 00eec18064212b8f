"""The command line front end (paper_1802_10453_b200/ffldl_b200),
mirroring the reference CLI's subcommands and exit codes (proj/tools/ffldl_main.cpp:20-25,
172-262).  Usage and parse paths run on the CPU; gen/factor/verify/bench need the GPU."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1802_10453_b200", "ffldl_b200")


def run(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, env=e)


def test_cli_usage_and_parse_errors(tmp_path):
    assert os.path.exists(CLI), "build the CLI (python -m paper_1802_10453_b200.build)"
    assert run().returncode == 2
    assert run("frobnicate").returncode == 2
    assert run("factor").returncode == 2  # -i required
    bad = tmp_path / "bad.txt"
    bad.write_text("SymMat 2 7\n0 1\n0 0\n")
    r = run("factor", "-i", bad)
    assert r.returncode == 4 and "not symmetric" in r.stderr
    assert run("factor", "-i", tmp_path / "missing").returncode == 4
    good = tmp_path / "good.txt"
    good.write_text("SymMat 2 7\n0 0\n0 3\n")
    assert run("factor", "-i", good, env={"RPM_LDLT_THRESHOLD": "x1"}).returncode == 2
    assert run("verify", "-i", good).returncode == 2  # -f required


@pytest.mark.gpu
def test_cli_gen_factor_verify_bench(gpu, oracle, tmp_path):
    import paper_1802_10453_b200 as ffb
    for kind, p, binary in (("config5", 131, True), ("hollow", 131, False), ("config3", 8388593, True),
                            ("rpm-half", 2, False)):
        m, f = tmp_path / f"{kind}.m", tmp_path / f"{kind}.f"
        g = ["--binary"] if binary else []
        assert run("gen", "--kind", kind, "-n", 200, "--modulus", p, "--seed", 9, "-o", m, *g).returncode == 0
        r = run("factor", "-i", m, "-o", f, *g)
        assert r.returncode == 0, r.stderr
        a, pp, sym = ffb.read_matrix(str(m))
        assert pp == p and sym
        got = ffb.read_factorization(str(f))
        want = oracle.ldlt(p, a)
        kd, val, val2 = got.diag.columns()
        assert got.rank == want.rank and np.array_equal(got.lower, want.lower)
        assert np.array_equal(got.perm.image_array(), want.perm) and np.array_equal(kd, want.dkind)
        r = run("verify", "-i", m, "-f", f, "--check-rpm")
        assert r.returncode == 0 and "rank profile matrix revealed" in r.stdout, r.stdout + r.stderr
        # a corrupted L entry is caught (exit 1)
        got.lower[-1, 0] = (got.lower[-1, 0] + 1) % p
        ffb.write_factorization(str(f) + "x", got)
        assert run("verify", "-i", m, "-f", str(f) + "x").returncode == 1
    r = run("factor", "-i", tmp_path / "config5.m", "--variant", "crout", "--threshold", 8)
    assert r.returncode == 0 and r.stdout.startswith("Factorization 200 131")
    r = run("bench", "--kind", "config5", "-n", 256, 512, "--modulus", 131)
    lines = r.stdout.strip().splitlines()
    assert r.returncode == 0 and lines[0] == "n,r,field,variant,seconds,mul_count,effective_gfops"
    assert [l.split(",")[:4] for l in lines[1:]] == [["256", "128", "131", "Cascade"], ["512", "256", "131", "Cascade"]]
