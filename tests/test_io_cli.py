"""The .tens format, JSON run config and CLI against bytes
and configs produced by the reference (tests/golden/make_golden.py gen_tens).
CPU-only except the end-to-end CLI reconstruction."""

import json

import numpy as np
import pytest

import paper_2301_03047_b200 as G
from paper_2301_03047_b200 import cli, config, tensorio
from conftest import load_golden


def test_tens_bytes_identical_to_reference(tmp_path):
    g = load_golden("tens")
    for i in range(int(g["n"])):
        a = g[f"arr{i}"]
        G.write_tensor(tmp_path / "t.tens", a)
        assert (tmp_path / "t.tens").read_bytes() == g[f"bytes{i}"].tobytes(), i
        got = G.read_tensor(tmp_path / "t.tens")
        want = g[f"read{i}"]
        assert got.dtype == want.dtype and np.array_equal(got, want), i
        pinned = G.read_tensor(tmp_path / "t.tens", pinned=True)
        assert np.array_equal(pinned, want)


def test_tens_u8_scaling_and_meta(tmp_path):
    a = np.arange(6, dtype=np.uint8).reshape(2, 3) * 51
    G.write_tensor(tmp_path / "u.tens", a)
    t, meta = G.read_tensor(tmp_path / "u.tens", with_meta=True)
    assert meta == {"peak": 255.0, "dtype_code": 3}
    assert np.array_equal(t, a / 255.0)
    raw = G.read_tensor(tmp_path / "u.tens", scale_u8=False)
    assert raw.dtype == np.uint8 and np.array_equal(raw, a)


def test_tens_errors(tmp_path):
    p = tmp_path / "bad.tens"
    p.write_bytes(b"NOTMAGIC" + bytes(8))
    with pytest.raises(tensorio.BadMagicError):
        G.read_tensor(p)
    G.write_tensor(p, np.zeros((4, 4)))
    p.write_bytes(p.read_bytes()[:-3])
    with pytest.raises(tensorio.TruncatedPayloadError):
        G.read_tensor(p)
    raw = bytearray(tensorio.MAGIC + (1).to_bytes(4, "little") + (2).to_bytes(4, "little")
                    + bytes([9]) + bytes(16))
    p.write_bytes(bytes(raw))
    with pytest.raises(tensorio.UnknownDtypeError):
        G.read_tensor(p)
    with pytest.raises(tensorio.UnknownDtypeError):
        G.write_tensor(p, np.zeros(3, dtype=np.int16))
    (tmp_path / "tile.txt").write_text("# tile\n0 1\n2\n")
    with pytest.raises(G.TensorFileError):
        tensorio.read_tile_file(tmp_path / "tile.txt")
    (tmp_path / "tile.txt").write_text("0 1\n\n2 3\n")
    assert tensorio.read_tile_file(tmp_path / "tile.txt").tolist() == [[0, 1], [2, 3]]


def test_run_config_matches_reference_serialization():
    g = load_golden("tens")
    ref_json = str(g["config_json"])
    run = config.parse_run_config(ref_json)
    assert run.solver.max_iters == 7 and run.solver.regularizer == "nlr-bm"
    assert run.solver.match.patch_size == 6 and run.solver.match.bm_window == 9
    assert run.operator.kind == "msfa" and run.operator.channels == 4
    assert json.loads(config.serialize_run_config(run)) == json.loads(ref_json)


@pytest.mark.parametrize("doc,frag", [
    ("{", "invalid JSON"), ("[]", "top level"), ({"solvr": {}}, "unknown keys"),
    ({"solver": {"max_iter": 3}}, "solver: unknown keys"),
    ({"solver": {"match": {"patchsize": 3}}}, "solver.match: unknown keys"),
    ({"solver": {"max_iters": 0}}, "max_iters"), ({"operator": 3}, "expected an object"),
])
def test_run_config_errors(doc, frag):
    with pytest.raises(config.ConfigError, match=frag):
        config.parse_run_config(doc)


def test_cli_exit_codes(tmp_path, capsys):
    assert cli.main(["demo", "--scene", "nope", "--out", str(tmp_path / "s.tens")]) == 2
    assert cli.main(["demo", "--scene", "cacti-blobs", "--height", "40", "--width", "36",
                     "--frames", "3", "--out", str(tmp_path / "s.tens")]) == 0
    assert G.read_tensor(tmp_path / "s.tens").shape == (40, 36, 3)
    assert cli.main(["mask", "gen", "--kind", "msfa", "--height", "8", "--width", "8",
                     "--channels", "4", "--msfa-kind", "bayer-like-2x2",
                     "--out", str(tmp_path / "m.tens")]) == 0
    assert G.read_tensor(tmp_path / "m.tens").shape == (8, 8, 4)
    (tmp_path / "bad.json").write_text('{"solver": {"bogus": 1}}')
    assert cli.main(["reconstruct", "--config", str(tmp_path / "bad.json"), "--measurement",
                     str(tmp_path / "s.tens"), "--out", str(tmp_path / "x.tens")]) == 2
    assert cli.main(["no-such-command"]) == 2


@pytest.mark.gpu
def test_cli_reconstruct_end_to_end(tmp_path):
    """demo -> simulate -> reconstruct on the device; the result equals the
    library call on the same inputs (bit-for-bit: same deterministic path)."""
    d = str(tmp_path)
    assert cli.main(["demo", "--scene", "cacti-blobs", "--height", "48", "--width", "40",
                     "--frames", "4", "--out", f"{d}/s.tens"]) == 0
    assert cli.main(["simulate", "--model", "cacti", "--scene", f"{d}/s.tens", "--out",
                     f"{d}/y.tens", "--save-mask", f"{d}/m.tens"]) == 0
    cfg = {"solver": {"max_iters": 6, "match": {"patch_size": 8, "group_size": 16,
                                                 "max_corners": 24, "exemplar_stride": 6}},
           "operator": {"kind": "cacti", "mask_path": f"{d}/m.tens"}}
    (tmp_path / "run.json").write_text(json.dumps(cfg))
    assert cli.main(["reconstruct", "--config", f"{d}/run.json", "--measurement",
                     f"{d}/y.tens", "--ref", f"{d}/s.tens", "--out", f"{d}/x.tens",
                     "--report", f"{d}/r.csv"]) == 0
    x = G.read_tensor(f"{d}/x.tens")
    run = config.parse_run_config(json.dumps(cfg))
    xl, rep = G.solve(run.operator.build(), G.read_tensor(f"{d}/y.tens"), run.solver,
                      ref=G.read_tensor(f"{d}/s.tens"))
    assert np.array_equal(x, xl)
    assert (tmp_path / "r.csv").read_text().startswith("iteration,residual")
    assert cli.main(["bench", "--sizes", "64", "--channels", "1,3", "--repeats", "1",
                     "--exemplars", "32", "--out", f"{d}/b.csv"]) == 0
    rows = (tmp_path / "b.csv").read_text().splitlines()
    assert rows[0].startswith("mode,height") and len(rows) == 5
