"""Data / result file formats against files written by the
reference's own data.py (tests/golden/make_golden.py formats()): the readers
return what the reference's readers return, the writers reproduce the
reference's files byte for byte, errors name the line, and the binary
latent sidecar round-trips."""
import math
import os

import numpy as np
import pytest

import paper_1603_08114_b200 as P
from conftest import golden

HERE = os.path.dirname(os.path.abspath(__file__))
FMT = os.path.join(HERE, "golden", "formats")
Z = golden("formats.npz")


def _read(path):
    with open(path, "rb") as fh:
        return fh.read()


def test_dataset_reads_and_writes_like_the_reference(tmp_path):
    ds = P.load_dataset(os.path.join(FMT, "dataset.csv"))
    assert np.array_equal(ds.returns, Z["returns"]) and np.array_equal(ds.rv, Z["rv"])
    assert np.array_equal(ds.log_rv, Z["log_rv"])
    assert ds.dates[0] == "2000-01-03" and len(ds.dates) == 40
    out = tmp_path / "d.csv"
    P.save_dataset(P.Dataset(returns=Z["returns"], rv=Z["rv"]), out)  # dates synthesized as the reference does
    assert _read(out) == _read(os.path.join(FMT, "dataset.csv"))


def test_truth_round_trip_and_bytes(tmp_path):
    params, h = P.load_truth(os.path.join(FMT, "truth.csv"))
    assert np.array_equal(h, Z["truth_h"])
    assert [params.phi, params.mu, params.xi, params.sigma_eta_sq, params.sigma_u_sq] == list(Z["truth_params"])
    tr = P.simulate_rsv(P.Params(0.97, -9.0, -0.3, 0.05, 0.1), 40, seed=3)
    out = tmp_path / "t.csv"
    P.save_truth(tr, out)
    assert _read(out) == _read(os.path.join(FMT, "truth.csv"))


def test_chain_with_latent_companion(tmp_path):
    ch = P.load_chain(os.path.join(FMT, "chain.csv"))
    assert np.array_equal(ch.mu, Z["chain_mu"]) and np.array_equal(ch.accept, Z["chain_accept"])
    assert np.array_equal(ch.delta_h, Z["chain_dh"]) and math.isinf(ch.delta_h[np.isinf(Z["chain_dh"])][0])
    assert np.array_equal(ch.latent, Z["chain_latent"])
    out = tmp_path / "c.csv"
    P.save_chain(ch, out)
    assert _read(out) == _read(os.path.join(FMT, "chain.csv"))
    assert _read(tmp_path / "c.latent.csv") == _read(os.path.join(FMT, "chain.latent.csv"))
    nolat = P.load_chain(os.path.join(FMT, "chain_nolatent.csv"))
    assert nolat.latent is None


def test_chain_binary_sidecar(tmp_path):
    ch = P.load_chain(os.path.join(FMT, "chain.csv"))
    out = tmp_path / "big.csv"
    P.save_chain(ch, out, latent="npy")
    assert (tmp_path / "big.latent.npy").exists() and not (tmp_path / "big.latent.csv").exists()
    back = P.load_chain(out)
    assert np.array_equal(back.latent, ch.latent) and np.array_equal(back.iters, ch.iters)
    with pytest.raises(ValueError):
        P.save_chain(ch, out, latent="parquet")


def test_intraday_and_rv_floor():
    panel = P.load_intraday(os.path.join(FMT, "intraday.csv"))
    assert panel.n_days == 3 and panel.dates == ["2000-01-03", "2000-01-04", "2000-01-05"]
    assert np.array_equal(P.compute_rv(panel), Z["intraday_rv"])
    assert P.compute_rv(panel)[2] == 1e-12


@pytest.mark.parametrize("text,msg", [
    ("date,return,rv\n2000-01-03,0.1,0.2\n", "at least 2 rows"),
    ("date,ret,rv\n2000-01-03,0.1,0.2\n", "expected header"),
    ("date,return,rv\n2000-01-03,0.1,0.2\n2000-01-04,0.1,-1\n", "line 3: rv=-1 is not positive"),
    ("date,return,rv\n2000-01-03,0.1,0.2\n2000-01-04,abc,0.1\n", "line 3: cannot parse return"),
    ("date,return,rv\n2000-01-03,0.1\n", "line 2: expected 3 columns"),
    ("# only a comment\n\n", "no header row"),
    ("date,return,rv\n", "empty dataset"),
])
def test_dataset_errors_name_the_line(tmp_path, text, msg):
    f = tmp_path / "bad.csv"
    f.write_text(text)
    with pytest.raises(P.DataFormatError, match=msg):
        P.load_dataset(f)


def test_missing_file_and_companion_mismatch(tmp_path):
    with pytest.raises(P.DataFormatError, match="no such file"):
        P.load_dataset(tmp_path / "nope.csv")
    ch = P.load_chain(os.path.join(FMT, "chain.csv"))
    out = tmp_path / "c.csv"
    P.save_chain(ch, out)
    lines = (tmp_path / "c.latent.csv").read_text().splitlines()
    (tmp_path / "c.latent.csv").write_text("\n".join(lines[:-1]) + "\n")
    with pytest.raises(P.DataFormatError, match="latent rows"):
        P.load_chain(out)
