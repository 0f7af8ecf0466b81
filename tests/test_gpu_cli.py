"""The CLI front end tools/fastdeblur_b200: the reference's
subcommands, file formats and exit codes (tools/fastdeblur.cpp:349-453,
io.cpp:34-233) over the B200 C ABI.  Cases follow the reference's own
tests/test_cli.cpp (identity-PSF eigenvalues, hoc-cosine border eigenvalues,
periodic blur = circular convolution, true-extended crop, noise level and
seed determinism, deblur diagnostics and curves, compare, exit code 2, --dims,
PGM), with the numerical outputs checked against the compiled reference
library / the numpy restatement."""
import os
import subprocess

import numpy as np
import pytest

import fdoracle as O
from paper_0906_2704_b200 import workloads as W

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "fastdeblur_b200")


def run(*args):
    p = subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


def write_signal(path, v):
    with open(path, "w") as f:
        for x in np.asarray(v).ravel():
            f.write(repr(float(x)) + "\n")
    return path


def read_signal(path):
    return np.array([float(s) for s in open(path).read().split() if not s.startswith("#")])


def write_psf(path, w):
    w = np.atleast_2d(np.asarray(w, dtype=np.float64))
    with open(path, "w") as f:
        f.write(f"{w.shape[0]} {w.shape[1]} {(w.shape[0] + 1) // 2} {(w.shape[1] + 1) // 2}\n")
        for row in w:
            f.write(" ".join(repr(float(x)) for x in row) + "\n")
    return path


def read_csv(path):
    lines = open(path).read().strip().split("\n")
    return lines[0], [ln.split(",") for ln in lines[1:]]


@pytest.fixture(scope="module", autouse=True)
def _binary():
    if not os.path.exists(BIN):
        pytest.skip("tools/fastdeblur_b200 not built (make -C tools)")


def test_eigs_identity_and_hoc_cosine(tmp_path):
    ident = write_psf(tmp_path / "id.txt", [1.0])
    out = tmp_path / "eigs.csv"
    assert run("eigs", "--psf", ident, "--n", 8, "--bc", "reflective", "--out", out)[0] == 0
    head, rows = read_csv(out)
    assert head == "index,real,imag" and len(rows) == 8
    for i, r in enumerate(rows):
        assert (int(r[0]), float(r[1]), float(r[2])) == (i + 1, 1.0, 0.0)
    p121 = write_psf(tmp_path / "psf.txt", [0.25, 0.5, 0.25])
    assert run("eigs", "--psf", p121, "--n", 10, "--bc", "hoc-cosine", "--out", out)[0] == 0
    _, rows = read_csv(out)
    assert float(rows[0][1]) == 1.0 and float(rows[-1][1]) == 1.0
    want = O.operator_eigenvalues(O.make_psf([0.25, 0.5, 0.25]), 10, O.HOC_COSINE)
    assert np.max(np.abs(np.array([float(r[1]) for r in rows]) - want.real)) < 1e-14
    assert run("eigs", "--psf", p121, "--n", 4, "--bc", "periodic", "--out", out)[0] == 0
    _, rows = read_csv(out)  # symbol of (1/4, 1/2, 1/4) at 2 pi k / 4
    assert np.allclose([float(r[1]) for r in rows], [1.0, 0.5, 0.0, 0.5], atol=1e-15)


def test_blur_periodic_true_extended_noise_and_seed(tmp_path, rng):
    p121 = write_psf(tmp_path / "psf.txt", [0.25, 0.5, 0.25])
    x = rng.standard_normal(16)
    inp = write_signal(tmp_path / "x.csv", x)
    out = tmp_path / "y.csv"
    assert run("blur", "--input", inp, "--psf", p121, "--bc", "periodic", "--output", out)[0] == 0
    want = 0.25 * np.roll(x, 1) + 0.5 * x + 0.25 * np.roll(x, -1)
    assert np.max(np.abs(read_signal(out) - want)) < 1e-14
    assert run("blur", "--input", inp, "--psf", p121, "--output", out)[0] == 0  # true-extended
    y = read_signal(out)
    assert y.shape == (14,)
    assert np.max(np.abs(y - W.convolve_valid(x, np.array([0.25, 0.5, 0.25])))) < 1e-15
    # noise: exactly the requested relative level, byte-identical for equal seeds
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    args = ["blur", "--input", inp, "--psf", p121, "--noise", 0.05, "--seed", 7]
    assert run(*args, "--output", a)[0] == 0 and run(*args, "--output", b)[0] == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    noisy = read_signal(a)
    assert abs(np.linalg.norm(noisy - y) / np.linalg.norm(y) - 0.05) < 1e-12
    assert np.max(np.abs(noisy - W.add_noise(y, 0.05, np.uint64(7)))) < 1e-13


def test_deblur_gcv_curves_and_reference(tmp_path):
    import reflib as R
    n, m = 64, 4
    psfw = W.gaussian_weights(m, 1.5)
    psf = write_psf(tmp_path / "gauss.txt", psfw)
    t = (np.arange(n + 2 * m) - m) / n
    fext = 1.0 + t + 0.8 * np.exp(-((t - 0.5) / 0.1) ** 2)
    obs = W.add_noise(W.convolve_valid(fext, psfw), 1e-3, np.uint64(3))
    truth = fext[m:m + n]
    inp, tr = write_signal(tmp_path / "obs.csv", obs), write_signal(tmp_path / "truth.csv", truth)
    out, curves = tmp_path / "restored.csv", tmp_path / "curves.csv"
    rc, so, se = run("deblur", "--input", inp, "--psf", psf, "--bc", "hoc-cosine", "--reg",
                     "laplacian", "--mu", "gcv", "--truth", tr, "--output", out, "--curves",
                     curves, "--mu-count", 60)
    assert rc == 0, se
    assert "source=gcv" in so and "rre=" in so
    head, rows = read_csv(curves)
    assert head == "mu,G,rre" and len(rows) == 60 and all(len(r) == 3 for r in rows)
    f = read_signal(out)
    mu = float(so.split("mu=")[1].split()[0])
    if R.available():  # the reference's deblur on the same file contents
        rf, rmu, rcurve, _ = R.deblur_1d(psfw, n, O.HOC_COSINE, 1, read_signal(inp), True,
                                         mu_min=1e-12, mu_max=10.0, count=60, want_curve=True)
        assert abs(mu / rmu[0] - 1) < 1e-10
        assert np.linalg.norm(f - rf[0]) / np.linalg.norm(rf[0]) < 1e-10
        G = np.array([float(r[1]) for r in rows])
        assert np.max(np.abs(G / rcurve[0] - 1)) < 1e-9
    # fixed mu, identity psf: returns the input; hoc-fourier prints the residue line
    ident = write_psf(tmp_path / "id.txt", [1.0])
    rc, so, _ = run("deblur", "--input", inp, "--psf", ident, "--bc", "hoc-fourier", "--mu", 1e-14,
                    "--output", out)
    assert rc == 0 and "source=fixed" in so and "imag_residue=" in so
    assert np.max(np.abs(read_signal(out) - obs)) < 1e-9


def test_compare_identity_and_exit_codes(tmp_path, rng):
    ident = write_psf(tmp_path / "id.txt", [1.0])
    x = np.cumsum(rng.standard_normal(40)) / 5 + 2.0
    inp = write_signal(tmp_path / "x.csv", x)
    out = tmp_path / "cmp.csv"
    rc, _, se = run("compare", "--input", inp, "--psf", ident, "--bc-list",
                    "periodic,reflective,antireflective,hoc-cosine,hoc-fourier", "--out", out,
                    "--mu-lo", 1e-14, "--mu-hi", 1e-8, "--mu-count", 8)
    assert rc == 0, se
    head, rows = read_csv(out)
    assert head == "bc,min_rre,mu_opt,mu_gcv,rre_gcv" and len(rows) == 5
    assert all(float(r[1]) <= 1e-10 for r in rows)
    # validation failures: exit code 2 (unknown bc, even psf, missing file, bad mu, no subcommand)
    assert run("eigs", "--psf", ident, "--n", 8, "--bc", "nope", "--out", out)[0] == 2
    bad = tmp_path / "bad.txt"
    bad.write_text("1 2 1 1\n0.5 0.5\n")
    assert run("eigs", "--psf", bad, "--n", 8, "--bc", "periodic", "--out", out)[0] == 2
    assert run("blur", "--input", tmp_path / "missing.csv", "--psf", ident, "--output", out)[0] == 2
    assert run("deblur", "--input", inp, "--psf", ident, "--bc", "periodic", "--mu", "-1",
               "--output", out)[0] == 2
    assert run()[0] == 2 and run("deblur")[0] == 2
    un = write_psf(tmp_path / "un.txt", [0.3, 0.5, 0.3])  # sums to 1.1: needs --normalize
    assert run("eigs", "--psf", un, "--n", 8, "--bc", "periodic", "--out", out)[0] == 2
    assert run("--normalize", "eigs", "--psf", un, "--n", 8, "--bc", "periodic", "--out", out)[0] == 0


def test_2d_dims_and_pgm(tmp_path, rng):
    w2 = np.outer(W.gaussian_weights(2, 1.0), W.gaussian_weights(1, 0.8))
    w2 /= w2.sum()
    psf = write_psf(tmp_path / "psf2.txt", w2)
    img = rng.random((20, 17))
    inp = write_signal(tmp_path / "img.csv", img)
    out = tmp_path / "blur.csv"
    assert run("blur", "--input", inp, "--psf", psf, "--dims", "20x17", "--output", out)[0] == 0
    y = read_signal(out)
    assert y.shape == (16 * 15,)
    want = np.zeros((16, 15))
    for j in range(5):
        for l in range(3):
            want += w2[j, l] * img[j:j + 16, l:l + 15]
    assert np.max(np.abs(y.reshape(16, 15) - want)) < 1e-15
    eigs = tmp_path / "e.csv"
    assert run("eigs", "--psf", psf, "--n", 9, "--n2", 7, "--bc", "reflective", "--out", eigs)[0] == 0
    assert len(read_csv(eigs)[1]) == 63
    # PGM in, P5 out with the source maxval; the 2D pipeline restores it
    pix = (rng.random((12, 14)) * 255).astype(np.uint8)
    pgm = tmp_path / "in.pgm"
    with open(pgm, "wb") as f:
        f.write(b"P5\n# comment\n14 12\n255\n" + pix.tobytes())
    ident = write_psf(tmp_path / "id.txt", [1.0])
    outp = tmp_path / "out.pgm"
    rc, so, se = run("deblur", "--input", pgm, "--psf", ident, "--bc", "hoc-cosine", "--mu", 1e-12,
                     "--output", outp)
    assert rc == 0, se
    data = open(outp, "rb").read()
    assert data.startswith(b"P5\n14 12\n255\n")
    assert np.array_equal(np.frombuffer(data[len(b"P5\n14 12\n255\n"):], np.uint8).reshape(12, 14), pix)
    cmp_out = tmp_path / "cmp2.csv"
    ext = write_signal(tmp_path / "ext.csv", rng.random((24, 21)) + 1.0)
    rc, _, se = run("compare", "--input", ext, "--psf", psf, "--dims", "24x21", "--noise", 0.01,
                    "--seed", 5, "--bc-list", "reflective,hoc-cosine", "--reg", "laplacian", "--out",
                    cmp_out, "--mu-count", 12)
    assert rc == 0, se
    assert len(read_csv(cmp_out)[1]) == 2
