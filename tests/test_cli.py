"""`solver` CLI above the C-ABI: census layout of PAPER Table 1,
RunConfig errors -> exit 1, run -> history CSV + summary, exit 0/2."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2312_10615_b200 as smg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2312_10615_b200", "solver")


def run(args, cfg=None, tmp=None):
    path = None
    if cfg is not None:
        path = os.path.join(tmp, "cfg.json")
        with open(path, "w") as f:
            f.write(cfg if isinstance(cfg, str) else json.dumps(cfg))
    return subprocess.run([CLI] + args + ([path] if path else []), capture_output=True, text=True, timeout=600)


def test_census_table1(tmp_path):
    r = run(["census"], {"nx": 128, "band_width": 1}, str(tmp_path))
    assert r.returncode == 0 and r.stdout.strip() == "8339456 385580 4.62%"
    n = smg.lib().smg_census(smg.GridDesc(3, 32, 32, 32, 1 / 32), 1, None)
    assert n == 32 ** 3 + 3 * 32 * 32 * 31


@pytest.mark.parametrize("cfg", ['{"nx": ', '{"ny": 8}', "not json"])
def test_malformed_config_exit_1(tmp_path, cfg):
    assert run(["census"], cfg, str(tmp_path)).returncode == 1


def test_usage_exit_1():
    assert subprocess.run([CLI], capture_output=True).returncode == 1


@pytest.mark.gpu
def test_run_writes_csv_and_summary(tmp_path):
    cfg = {"nx": 32, "levels": 3, "eta": 1.0, "tol": 1e-6, "seed": 0, "output_dir": str(tmp_path)}
    r = run(["run"], cfg, str(tmp_path))
    assert r.returncode == 0, r.stderr
    rows = open(tmp_path / "history_mg-sqmr.csv").read().splitlines()
    assert rows[0] == "iteration,rel_residual,seconds"
    h = np.array([float(x.split(",")[1]) for x in rows[1:]])
    s = smg.Solver(32, levels=3, eta=1.0)
    _, hp, _, _ = s.sqmr(smg.forcing(32, seed=0), 1e-6, 200)
    assert np.array_equal(h, hp)  # same path, %.17g round-trips
    summ = dict(l.split(": ") for l in open(tmp_path / "summary.txt").read().splitlines())
    assert summ["status"] == "converged" and int(summ["iterations"]) == len(h)
    assert float(summ["div_u_inf"]) < 1e-6
    cfg.update(method="mg", maxit=2, tol=1e-12)
    r = run(["run"], cfg, str(tmp_path))
    assert r.returncode == 2  # not converged
    assert len(open(tmp_path / "history_mg.csv").read().splitlines()) == 3


@pytest.mark.gpu
def test_run_writes_vtk_fields(tmp_path):
    """emit flag vtk: legacy ASCII structured points, pressure + cell-centred velocity."""
    cfg = {"nx": 16, "ny": 8, "nz": 12, "h": 1 / 8, "levels": 2, "eta": 1.0, "tol": 1e-8, "seed": 3,
           "vtk": 1, "output_dir": str(tmp_path)}
    r = run(["run"], cfg, str(tmp_path))
    assert r.returncode == 0, r.stderr
    lines = open(tmp_path / "fields.vtk").read().splitlines()
    assert lines[0].startswith("# vtk DataFile") and lines[2] == "ASCII"
    assert "DIMENSIONS 17 9 13" in lines and "CELL_DATA 1536" in lines
    i = lines.index("LOOKUP_TABLE default")
    p = np.array([float(v) for v in lines[i + 1:i + 1 + 1536]])
    j = lines.index("VECTORS velocity double")
    vel = np.array([[float(t) for t in l.split()] for l in lines[j + 1:j + 1 + 1536]])
    s = smg.Solver(16, 8, 12, h=1 / 8, levels=2, eta=1.0)
    x, _, _, _ = s.sqmr(smg.forcing(16, 8, 12, h=1 / 8, seed=3), 1e-8, 200)
    nu, nv, nw = 15 * 8 * 12, 16 * 7 * 12, 16 * 8 * 11
    assert np.array_equal(p, x[nu + nv + nw:])  # %.17g round-trips doubles exactly
    u = np.zeros((12, 8, 17))
    u[:, :, 1:16] = x[:nu].reshape(12, 8, 15)
    assert np.allclose(vel[:, 0], (0.5 * (u[:, :, :-1] + u[:, :, 1:])).ravel(), rtol=0, atol=1e-15)
    s.close()


@pytest.mark.gpu
def test_verify_symmetry():
    """`solver verify`: materialised GPU smoother and V-cycle maps symmetric < 1e-10."""
    r = subprocess.run([CLI, "verify", "--max-n", "8"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.splitlines()
    assert len(lines) == 15 and all(l.endswith("PASS") for l in lines)  # 2 sizes x 2 Vanka kinds x 3 maps + labelled


def test_verify_usage():
    assert subprocess.run([CLI, "verify", "--max-n"], capture_output=True).returncode == 1


def _domain(tmp_path):
    from paper_2312_10615_b200 import scenarios
    lab = scenarios.cylinder3d(32, 16, 8)
    path = str(tmp_path / "cyl.dom")
    scenarios.write_domain_file(path, lab, 1 / 16)
    back, h = scenarios.read_domain_file(path)
    assert np.array_equal(back, lab) and h == 1 / 16
    return lab, path


def test_census_of_a_domain_file(tmp_path):
    """Domain file format of SPEC:88 (header `dim nx ny nz h`, one D / I / E character per cell)."""
    lab, path = _domain(tmp_path)
    r = run(["census"], {"domain": path, "band_width": 1}, str(tmp_path))
    c = smg.census_labels(lab)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split()[:2] == [str(c["N"]), str(c["V1"])]
    open(path, "a").write("I")  # one label too many
    assert run(["census"], {"domain": path}, str(tmp_path)).returncode == 1
    open(path, "w").write("3 4 4 4 0.25\n" + "IIXI" * 16)
    assert run(["census"], {"domain": path}, str(tmp_path)).returncode == 1
    assert run(["census"], {"domain": str(tmp_path / "missing.dom")}, str(tmp_path)).returncode == 1


@pytest.mark.gpu
def test_run_on_a_domain_file(tmp_path):
    lab, path = _domain(tmp_path)
    cfg = {"domain": path, "levels": 3, "eta": 1.0, "tol": 1e-8, "seed": 4, "forcing": "channel",
           "output_dir": str(tmp_path)}
    r = run(["run"], cfg, str(tmp_path))
    assert r.returncode == 0, r.stderr
    rows = open(tmp_path / "history_mg-sqmr.csv").read().splitlines()
    h = np.array([float(x.split(",")[1]) for x in rows[1:]])
    s = smg.Solver.from_labels(lab, h=1 / 16, levels=3)
    _, hp, _, st = s.sqmr(smg.forcing_labels(lab, 1 / 16, smg.FORCE_CHANNEL, 4), 1e-8, 200)
    s.close()
    assert st == smg.SMG_CONVERGED and np.array_equal(h, hp)
    summ = dict(l.split(": ") for l in open(tmp_path / "summary.txt").read().splitlines())
    assert summ["status"] == "converged" and int(summ["dof"]) == smg.census_labels(lab)["N"]


@pytest.mark.gpu
def test_matrix_market_export(tmp_path):
    """`solver matrix`: the fine-level L materialised through the GPU operator as
    Matrix Market coordinate text: equals the oracle's dense L and is symmetric."""
    import oracle
    _, path = _domain(tmp_path)
    from paper_2312_10615_b200 import scenarios
    lab = scenarios.cylinder3d(16, 8, 8, cx=0.4, cy=0.5, radius=0.2)
    scenarios.write_domain_file(path, lab, 1 / 8)
    r = run(["matrix"], {"domain": path, "levels": 2, "eta": 1.0}, str(tmp_path))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general"
    n, n2, nnz = (int(v) for v in lines[1].split())
    A = np.zeros((n, n))
    for l in lines[2:]:
        i, j, v = l.split()
        A[int(i) - 1, int(j) - 1] = float(v)
    assert n == n2 and len(lines) == 2 + nnz
    o = oracle.Oracle(0, levels=2, labels=lab, h=1 / 8)
    assert np.array_equal(A, o.dense(0, False))
    assert np.abs(A - A.T).max() <= 1e-12 * np.abs(A).max()
    big = run(["matrix"], {"nx": 16, "levels": 2}, str(tmp_path))
    assert big.returncode == 1  # N above the dense cap
