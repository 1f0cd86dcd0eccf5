"""The app/CLI layer: readers, discretisation, exports and
exit codes on CPU; solves on the GPU."""
import json
import os

import numpy as np
import pytest

from paper_1810_00118_b200 import cli, instances


def test_pgm_p2_p5_roundtrip(tmp_path):
    img = np.arange(12, dtype=np.float64).reshape(3, 4) * 1000
    p5 = tmp_path / "a.pgm"
    cli.write_pgm(str(p5), img)
    back = cli.read_pgm(str(p5))
    assert back.shape == (3, 4)
    np.testing.assert_allclose(back / back.max(), img / img.max(), atol=1e-4)
    p2 = tmp_path / "b.pgm"
    p2.write_text("P2\n# a comment\n3 2\n255\n0 1 2\n3 4 255\n")
    assert cli.read_pgm(str(p2)).tolist() == [[0, 1, 2], [3, 4, 255]]


def test_bad_inputs_are_format_errors(tmp_path):
    bad = tmp_path / "x.pgm"
    bad.write_bytes(b"P9\n1 1\n255\n\x00")
    with pytest.raises(cli.FormatError):
        cli.read_image(str(bad))
    rag = tmp_path / "r.csv"
    rag.write_text("1,2\n3\n")
    with pytest.raises(cli.FormatError):
        cli.read_image(str(rag))
    rect = tmp_path / "q.csv"
    rect.write_text("1,2,3\n4,5,6\n")
    with pytest.raises(cli.FormatError, match="square"):
        cli.read_image(str(rect))
    zero = tmp_path / "z.csv"
    zero.write_text("0,0\n0,0\n")
    with pytest.raises(cli.FormatError, match="all-zero"):
        cli.read_image(str(zero))
    assert cli.main(["solve", "--a", str(bad), "--b", str(bad)]) == cli.EXIT_FORMAT
    assert cli.main(["nonsense"]) == cli.EXIT_USAGE


def test_discretize_spec_examples():
    """pixel centres on [0,1]^2 (an M x M image resampled
    onto M nodes is the image itself, scaled), unit mass in the L1_h sense,
    constant image -> constant field, checkerboard 64 -> N = 32 mass 1 to 1e-12,
    corner pixels on corner nodes."""
    img = np.random.default_rng(0).random((17, 17)) + 0.1
    d = cli.discretize(img, 16)  # 17 nodes per side = the pixel lattice
    h = 1.0 / 16
    assert abs(d.sum() * h * h - 1.0) <= 1e-12
    np.testing.assert_allclose(d / d.sum(), img / img.sum(), rtol=1e-12)
    two = np.array([[1.0, 2.0], [3.0, 4.0]])
    np.testing.assert_allclose(cli.discretize(two, 1), two / 10.0, rtol=1e-15)
    const = cli.discretize(np.ones((8, 8)), 32)
    assert np.allclose(const, const[0, 0])
    cb = (np.indices((64, 64)).sum(axis=0) % 2).astype(float)
    assert abs(cli.discretize(cb, 32).sum() / 32 ** 2 - 1.0) <= 1e-12
    dirac = np.zeros((64, 64))
    dirac[0, 63] = 1.0
    dd = cli.discretize(dirac, 64)
    assert np.unravel_index(dd.argmax(), dd.shape) == (0, 64)


def test_field_csv_roundtrip_bit_exact(tmp_path):
    """17 significant digits re-import bit-exactly."""
    rng = np.random.default_rng(1)
    blocks = {"x_edges": rng.standard_normal((5, 4)), "y_edges": rng.standard_normal((4, 5))}
    p = tmp_path / "f.csv"
    cli.write_field_csv(str(p), blocks)
    back = cli.read_field_csv(str(p))
    for k in blocks:
        assert np.array_equal(back[k], blocks[k])


def test_gen_deterministic(tmp_path):
    a1, b1 = tmp_path / "a1.csv", tmp_path / "b1.csv"
    a2, b2 = tmp_path / "a2.csv", tmp_path / "b2.csv"
    for a, b in ((a1, b1), (a2, b2)):
        assert cli.main(["gen", "--kind", "two_blobs", "--n", "16", "--seed", "3",
                         "--out-a", str(a), "--out-b", str(b)]) == 0
    assert a1.read_text() == a2.read_text()


@pytest.mark.gpu
@pytest.mark.parametrize("p", ["1", "2", "inf"])
def test_cli_solve_dirac_pair(tmp_path, p):
    """SPEC.md:502 (and acceptance 2): dirac_pair corners ->
    distance 1 +- 1e-3.  The corner pixels land on the corner nodes
    (SPEC.md:468); the bilinear weight 1/n that leaks to the next node inward
    moves the transport length by ~2/n^2."""
    n = 64
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(["gen", "--kind", "dirac_pair", "--n", str(n), "--out-a", str(a),
                     "--out-b", str(b)]) == 0
    out = tmp_path / "r.json"
    rc = cli.main(["solve", "--a", str(a), "--b", str(b), "--p", p, "--algo", "pdhg",
                   "--tol", "1e-10", "--out", str(out), "--export-flux", str(tmp_path / "f.csv"),
                   "--export-potential", str(tmp_path / "p.csv")])
    rep = json.loads(out.read_text())
    assert rc == 0 and rep["converged"]
    assert abs(rep["distance"] - 1.0) <= 1e-3
    f = cli.read_field_csv(str(tmp_path / "f.csv"))
    assert f["x_edges"].shape == (n + 1, n)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["cp", "ml-cp", "ml-pdhg"])
def test_cli_solve_identical_images(tmp_path, algo):
    """identical inputs -> distance ~ 0."""
    a = tmp_path / "a.pgm"
    cli.write_pgm(str(a), instances.blurred_noise_image(0, m=64))
    out = tmp_path / "r.json"
    rc = cli.main(["solve", "--a", str(a), "--b", str(a), "--p", "2", "--algo", algo,
                   "--out", str(out)])
    rep = json.loads(out.read_text())
    assert rc == 0 and abs(rep["distance"]) <= 1e-9
    assert [l["h"] for l in rep["levels"]][-1] == 1.0 / 64
