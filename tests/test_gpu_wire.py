"""Device wire format (lags_wire_encode / lags_wire_decode) against the reference's bytes: the
golden chunk and message encodings (tests/golden/wire_cases.json, made by the reference's
encode_chunk / encode_message), its round-trip and truncation tests (R: tests/test_sparsify.py:
291-329), and bucket messages from a real compress."""

import struct

import numpy as np
import pytest
import torch

from conftest import load_json

pytestmark = pytest.mark.gpu

import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402


def chunk(layer_id, n, dim=64):
    return L.SparseChunk(layer_id, dim, np.arange(n, dtype=np.int64), np.arange(1.0, n + 1.0), k_target=max(n, 1))


def test_golden_chunks_bit_exact():
    for c in load_json("wire_cases.json")["chunks"]:
        ch = L.SparseChunk(c["layer_id"], c["dim"], np.array(c["idx"]), np.array(c["vals"]), k_target=len(c["idx"]))
        raw = L.encode_chunk(ch)
        assert raw.hex() == c["hex"]
        back, off = L.decode_chunk(raw)
        assert off == len(raw) and back.layer_id == c["layer_id"] and back.dim == c["dim"]
        assert back.indices.tolist() == c["idx"] and back.values.tolist() == c["vals"]
        assert back.values.dtype == np.float64 and back.k_target == len(c["idx"])
        assert L.encode_chunk(back) == raw


def test_golden_messages_bit_exact():
    n = 0
    for c in load_json("wire_cases.json")["flush"]:
        if c["hex"] is None:
            continue
        msg = L.fusion_flush([chunk(i + 1, k) for i, k in enumerate(c["counts"])], c["cap"], c["first"])
        raw = L.encode_message(msg)
        assert raw.hex() == c["hex"]
        back = L.decode_message(raw)
        assert [x.layer_id for x in back.chunks] == c["result"]
        assert L.encode_message(back) == raw
        n += 1
    assert n > 5


def test_reference_round_trip_and_sizes():
    rng = np.random.default_rng(10)
    for _ in range(30):
        x = rng.standard_normal(50)
        ch = L.top_k(x, int(rng.integers(1, 20)), layer_id=int(rng.integers(0, 9)))
        raw = L.encode_chunk(ch)
        back, off = L.decode_chunk(raw)
        assert off == len(raw)
        np.testing.assert_array_equal(back.indices, ch.indices)
        np.testing.assert_array_equal(back.values, ch.values)
    assert len(L.encode_chunk(chunk(3, 5))) == 12 + 5 * 12
    assert L.encode_message(L.FusionMessage(())) == b"\x00\x00\x00\x00"
    assert L.decode_message(b"\x00\x00\x00\x00").chunks == ()
    # fp32 values widen exactly; an empty chunk; decode_chunk at an offset
    c32 = L.SparseChunk(7, 10, np.array([1, 4]), np.array([0.1, -2.5], dtype=np.float32), k_target=3)
    raw = b"junk" + L.encode_chunk(c32) + L.encode_chunk(chunk(2, 0))
    back, off = L.decode_chunk(raw, 4)
    assert back.values.tolist() == [float(np.float32(0.1)), -2.5] and off == 4 + 36
    empty, end = L.decode_chunk(raw, off)
    assert len(empty) == 0 and end == len(raw)


def test_rejections_match_reference():
    raw = L.encode_chunk(chunk(1, 4))
    with pytest.raises(L.StructureError, match="truncated chunk payload"):
        L.decode_chunk(raw[:-3])
    with pytest.raises(L.StructureError, match="truncated chunk header"):
        L.decode_chunk(raw[:8])
    msg = L.encode_message(L.fusion_flush([chunk(1, 2)], 10**6, True))
    with pytest.raises(L.StructureError, match="1 trailing bytes"):
        L.decode_message(msg + b"\x00")
    with pytest.raises(L.StructureError, match="truncated message header"):
        L.decode_message(b"\x01\x00")
    with pytest.raises(L.StructureError, match="truncated chunk header"):
        L.decode_message(struct.pack("<I", 2) + L.encode_chunk(chunk(1, 2)))
    # invalid chunks: range is checked before order, and the first bad chunk wins
    bad_order = struct.pack("<III", 1, 64, 2) + struct.pack("<Id", 5, 1.0) + struct.pack("<Id", 3, 2.0)
    bad_range = struct.pack("<III", 2, 4, 2) + struct.pack("<Id", 5, 1.0) + struct.pack("<Id", 6, 2.0)
    with pytest.raises(L.StructureError, match="strictly increasing"):
        L.decode_chunk(bad_order)
    with pytest.raises(L.StructureError, match="out of range"):
        L.decode_chunk(bad_range)
    with pytest.raises(L.StructureError, match="strictly increasing"):
        L.decode_message(struct.pack("<I", 2) + bad_order + bad_range)
    with pytest.raises(L.StructureError, match="out of range"):
        L.decode_message(struct.pack("<I", 2) + bad_range + bad_order)


def test_bucket_message_encodes_like_the_reference():
    from paper_1911_08727_b200.workloads import resnet20

    dims = [p.numel() for p in resnet20().parameters()]
    ks = [max(1, d // 1000) for d in dims]
    b = L.Bucket(dims, ks, N.F32)
    gen = torch.Generator(device="cuda").manual_seed(5)
    n = sum(dims)
    r = torch.zeros(n, device="cuda")
    msg = b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        b.compress(torch.randn(n, device="cuda", generator=gen), r, 0.1, msg, st)
    ids = list(range(len(dims), 0, -1))  # any u32 ids, e.g. the reference's L..1 visiting order
    wire, wlen, err = b.encode_wire(msg, ids)
    assert int(err.item()) & (2**64 - 1) == N.WIRE_OK
    raw = wire[: int(wlen.item())].cpu().numpy().tobytes()
    chunks = [L.SparseChunk(i, d, ix, vx, k_target=k) for i, d, k, (ix, vx) in zip(ids, dims, ks, b.unpack(msg))]
    assert raw == L.encode_message(L.FusionMessage(tuple(chunks)))
    back = b.decode_wire(wire, int(wlen.item()), ids)
    for (i0, v0), (i1, v1) in zip(b.unpack(msg), b.unpack(back)):
        np.testing.assert_array_equal(i0, i1)
        np.testing.assert_array_equal(v0, v1)
    with pytest.raises(L.StructureError):
        b.decode_wire(wire, int(wlen.item()), list(range(1, len(dims) + 1)))
