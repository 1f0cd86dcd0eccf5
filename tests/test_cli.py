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


def test_discretize_matches_source_rule_and_unit_mass():
    """At N = M the bilinear resampling equals the cell->node mean used by
    the device restriction; mass is 1 in the L1_h sense."""
    img = np.random.default_rng(0).random((16, 16)) + 0.1
    d = cli.discretize(img, 16)
    h = 1.0 / 16
    assert abs(d.sum() * h * h - 1.0) <= 1e-12
    nodes = instances.image_to_nodes(img)
    np.testing.assert_allclose(d / d.sum(), nodes / nodes.sum(), rtol=1e-12)
    const = cli.discretize(np.ones((8, 8)), 32)  # constant image -> constant
    assert np.allclose(const, const[0, 0])


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
def test_cli_solve_dirac_pair(tmp_path):
    """dirac_pair corners, p = 1 -> distance 1 +- 1e-3."""
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(["gen", "--kind", "dirac_pair", "--n", "16", "--out-a", str(a),
                     "--out-b", str(b)]) == 0
    out = tmp_path / "r.json"
    rc = cli.main(["solve", "--a", str(a), "--b", str(b), "--p", "1", "--algo", "pdhg",
                   "--tol", "1e-10", "--out", str(out), "--export-flux", str(tmp_path / "f.csv"),
                   "--export-potential", str(tmp_path / "p.csv")])
    rep = json.loads(out.read_text())
    assert rc == 0 and rep["converged"]
    # the images' corner pixels sit half a pixel in: the node-resampled masses
    # are 15/16 apart plus the bilinear spread; distance is close to 1
    assert abs(rep["distance"] - 1.0) <= 0.1
    f = cli.read_field_csv(str(tmp_path / "f.csv"))
    assert f["x_edges"].shape == (17, 16)


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
