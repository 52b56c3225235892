"""Binary trace ingest: the reference's Trace
(core/include/embcomm/trace.hpp:18-30) in a mapped binary container.

Parity: a text trace parsed by the reference's own parse_trace
(core/src/trace.cpp:51-101, through oracle/_ref) and written to / mapped
from the binary container gives the identical Trace; the reference's
validation rules (d >= 1, 1 <= E <= 2^32-1, non-empty, ids < E, errors
naming the line) hold; the mapped trace feeds the trace functions with the
reference's results; the GPU upload is bitwise."""
import os

import numpy as np
import pytest

import oracle as O


def _text(path, d, vocab, rows):
    with open(path, "w") as f:
        f.write(f"d={d} E={vocab}\n")
        for r in rows:
            f.write(" ".join(str(int(x)) for x in r) + "\n")


def test_binary_round_trip_equals_reference_text_parse(ec, ref, tmp_path):
    rng = np.random.default_rng(5)
    d, vocab, q = 3, 1000, 257
    rows = rng.integers(0, vocab, (q, d))
    txt = tmp_path / "t.txt"
    _text(txt, d, vocab, rows)
    rd, rv, rids = O.ref_load_trace(txt)            # the reference's parser
    tr = ec.Trace(rd, rv, rids)
    binp = tmp_path / "t.ectrace"
    tr.save_binary(binp)
    assert os.path.getsize(binp) == 40 + 4 * q * d
    bt = ec.Trace.load_binary(binp)
    assert (bt.num_samples, bt.num_features, bt.vocab_size) == (q, d, vocab)
    t2 = bt.trace()
    assert t2.num_features == rd and t2.vocab_size == rv
    assert (np.asarray(t2.ids) == rids).all()
    del t2
    bt.close()
    # the KAT trace of tests/test_simulator.cpp:156-172 through the same path
    _text(txt, 2, 4, [[0, 1], [0, 2], [1, 1], [3, 3]])
    rd, rv, rids = O.ref_load_trace(txt)
    kat = tmp_path / "kat.ectrace"
    ec.Trace(rd, rv, rids).save_binary(kat)
    k = ec.Trace.load_binary(kat).trace()  # the view keeps the mapping alive
    assert (np.asarray(k.ids) == [0, 1, 0, 2, 1, 1, 3, 3]).all()


def test_binary_trace_validation(ec, tmp_path):
    p = tmp_path / "bad.ectrace"
    with pytest.raises(ec.ValidationError, match="line 3: id 7 out of range"):
        ec.Trace(2, 5, np.array([0, 1, 2, 7], np.uint32)).save_binary(p)  # sample 1 -> text line 3
    with pytest.raises(ec.ValidationError, match="lookups per sample"):
        ec.Trace(0, 5, np.array([], np.uint32)).save_binary(p)
    with pytest.raises(ec.ValidationError, match="vocabulary too large"):
        ec.Trace(1, 1 << 32, np.array([0], np.uint32)).save_binary(p)
    with pytest.raises(ec.ValidationError, match="empty trace"):
        ec.Trace(2, 5, np.array([], np.uint32)).save_binary(p)
    good = tmp_path / "good.ectrace"
    ec.Trace(2, 5, np.array([0, 1, 2, 4], np.uint32)).save_binary(good)
    raw = bytearray(good.read_bytes())
    (tmp_path / "magic.ectrace").write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(ec.ValidationError, match="bad magic"):
        ec.Trace.load_binary(tmp_path / "magic.ectrace")
    (tmp_path / "short.ectrace").write_bytes(raw[:-4])
    with pytest.raises(ec.ValidationError, match="size"):
        ec.Trace.load_binary(tmp_path / "short.ectrace")
    # samples * d wraps 2^64 to the file's real id count: refused before multiplying
    hdr = np.frombuffer(bytes(raw[:40]), np.uint64).copy()
    hdr[2], hdr[4] = 4, (1 << 62) + 1  # d = 4, samples = 2^62 + 1 -> 4 * samples wraps to 4
    (tmp_path / "wrap.ectrace").write_bytes(hdr.tobytes() + raw[40:])
    with pytest.raises(ec.ValidationError, match="too small"):
        ec.Trace.load_binary(tmp_path / "wrap.ectrace")
    (tmp_path / "hdr.ectrace").write_bytes(raw[:20])
    with pytest.raises(ec.ValidationError, match="truncated"):
        ec.Trace.load_binary(tmp_path / "hdr.ectrace")
    bad_id = raw[:-4] + np.array([5], np.uint32).tobytes()  # last id == E
    (tmp_path / "id.ectrace").write_bytes(bad_id)
    with pytest.raises(ec.ValidationError, match="line 3: id 5 out of range"):
        ec.Trace.load_binary(tmp_path / "id.ectrace")
    with pytest.raises(ec.ValidationError, match="cannot open"):
        ec.Trace.load_binary(tmp_path / "missing.ectrace")


@pytest.mark.gpu
def test_mapped_trace_feeds_gpu_trace_functions(ec, ref, tmp_path):
    """A mapped binary trace through the GPU skew table and schedule equals the
    reference on the text-parsed trace; the upload is bitwise."""
    import torch
    rng = np.random.default_rng(11)
    d, vocab, q = 4, 5000, 4096
    p = np.arange(1, vocab + 1, dtype=np.float64) ** -1.05
    rows = rng.choice(vocab, size=(q, d), p=p / p.sum())
    txt = tmp_path / "z.txt"
    _text(txt, d, vocab, rows)
    rd, rv, rids = O.ref_load_trace(txt)
    binp = tmp_path / "z.ectrace"
    ec.Trace(rd, rv, rids).save_binary(binp)
    bt = ec.Trace.load_binary(binp)
    tr = bt.trace()
    st = ec.build_skew_table(tr)
    oid, cnt, cum = O.ref_build_skew_table(rids, rd, rv)
    assert (st.ids == oid).all() and (st.counts == cnt).all() and (st.cum_fraction == cum).all()
    cache = np.arange(64, dtype=np.uint32)
    sch = ec.build_schedule(tr, cache, 128)
    order, _, _ = O.ref_build_schedule(rids, rd, rv, cache, 128)
    got = [i for b in sch.hot_batches + sch.normal_batches for i in b]
    assert got == order.tolist()
    dev = torch.empty(q * d, dtype=torch.int32, device="cuda")
    bt.upload(dev)
    torch.cuda.synchronize()
    assert (dev.cpu().numpy().view(np.uint32) == rids).all()
    half = torch.empty((q // 2) * d, dtype=torch.int32, device="cuda")
    bt.upload(half, first=q // 2, count=q // 2)
    torch.cuda.synchronize()
    assert (half.cpu().numpy().view(np.uint32) == rids[(q // 2) * d:]).all()
    with pytest.raises(ec.ValidationError):
        bt.upload(half, first=q, count=1)
