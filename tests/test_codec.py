"""Backup codec (native host code, csrc/codec.cpp) against the reference's
own payloads (tests/golden: resilience.encode run on the unmodified
reference) and the restated loop (oracle/codec.py).  Byte-exact.  CPU only
(the hierarchical codec, whose transfers run on the GPU, is in
test_gpu_multigrid.py)."""

import numpy as np
import pytest

import paper_1911_01492_b200 as pb
from paper_1911_01492_b200 import codec as cd
from oracle import codec as oc

NAMES = ("smooth", "random", "jumps", "ties", "adaptive", "empty")


@pytest.mark.parametrize("name", NAMES)
def test_payload_matches_reference_golden(golden, name):
    g = lambda k: golden[f"codec/{name}/{k}"]
    x, kind = g("x"), str(g("kind"))
    rn = float(g("rn"))
    codec = cd.Codec(kind, tau=float(g("tau")), c=float(g("c")))
    snap = cd.encode(codec, x, residual_norm=rn if rn > 0 else None)
    assert snap.tau_used == float(g("tau_used"))
    assert snap.payload == g("payload").tobytes()
    assert snap.n == x.size and snap.payload_len == g("payload").size
    dec = cd.decode(snap)
    assert np.array_equal(dec, g("decoded"))
    assert np.all(np.abs(dec - x) <= snap.tau_used)
    # the restatement agrees too (pins the oracle)
    assert oc.quantize(x, snap.tau_used) == snap.payload
    assert np.array_equal(oc.dequantize(snap.payload), dec)


def test_random_vectors_match_restatement():
    rng = np.random.default_rng(3)
    for n, tau, scale in ((2000, 1e-8, 1.0), (777, 0.25, 100.0), (64, 1e-300, 1.0),
                          (500, 1e200, 1e280)):
        x = rng.standard_normal(n) * scale
        x[::37] *= 1e12                           # escapes
        p = cd.quantize(x, tau)
        assert p == oc.quantize(x, tau)
        assert np.array_equal(cd.dequantize(p), oc.dequantize(p))


def test_codec_errors_and_kinds():
    with pytest.raises(cd.CodecError, match="unknown codec kind"):
        cd.Codec("lz4")
    with pytest.raises(cd.CodecError, match="tau must be positive"):
        cd.Codec("accuracy_bounded", tau=0.0)
    with pytest.raises(cd.CodecError, match="coupling factor"):
        cd.Codec("adaptive_accuracy", c=-1.0)
    with pytest.raises(cd.CodecError, match="needs a hierarchy"):
        cd.Codec("hierarchical")
    with pytest.raises(cd.CodecError, match="non-finite"):
        cd.encode(cd.Codec("accuracy_bounded"), np.array([1.0, np.nan]))
    with pytest.raises(cd.CodecError, match="positive residual norm"):
        cd.encode(cd.Codec("adaptive_accuracy"), np.ones(3))
    z = cd.encode(cd.Codec("zero"), np.ones(5), source_rank=2, iteration=7)
    assert z.payload_len == 8 and np.array_equal(cd.decode(z), np.zeros(5))
    assert (z.source_rank, z.iteration, z.uncompressed_len) == (2, 7, 40)
    with pytest.raises(cd.CodecError, match="truncated"):
        cd.dequantize(cd.quantize(np.arange(10.0) * 1e30, 1e-3)[:-3])


def test_encode_many_threads_match_single():
    rng = np.random.default_rng(5)
    segs = [rng.standard_normal(n) for n in (1000, 10, 0, 4096, 333)]
    codec = cd.Codec("adaptive_accuracy", c=0.5)
    norms = [1e-3, 2.0, 1.0, 1e-6, 0.1]
    many = cd.encode_many(codec, segs, norms, iteration=4, threads=3)
    for r, (x, s) in enumerate(zip(segs, many)):
        one = cd.encode(codec, x, residual_norm=norms[r], source_rank=r, iteration=4)
        assert s.payload == one.payload and s.source_rank == r and s.tau_used == one.tau_used
        assert np.array_equal(cd.decode(s), cd.decode(one))


def test_package_exports():
    for name in ("Codec", "BackupSnapshot", "CodecError", "encode", "decode", "CODEC_KINDS"):
        assert hasattr(pb, name)
