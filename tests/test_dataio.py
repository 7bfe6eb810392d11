"""Tensor I/O: the reference's JSON document codec (bc/dataio.py:89-106,
pkg/tests/test_dataio.py round trips) and the packed binary format."""

import json

import numpy as np
import pytest

from paper_1701_05420_b200 import BlockSymTensor, ValidationError
from paper_1701_05420_b200.dataio import emit_tensor, load_packed, load_tensor, save_packed
from paper_1701_05420_b200.layout import layout


def _tensor(n, m, b, rng):
    return BlockSymTensor.from_packed(n, m, b, rng.standard_normal(layout(n, m, b).size))


@pytest.mark.parametrize("n,m,b", [(5, 3, 2), (7, 4, 3), (4, 2, 5), (9, 1, 2)])
def test_json_roundtrip_bitwise(n, m, b, rng, tmp_path):
    t = _tensor(n, m, b, rng)
    p = tmp_path / "t.json"
    emit_tensor(t, p)
    back = load_tensor(p)
    assert (back.n, back.m, back.b) == (n, m, b)
    np.testing.assert_array_equal(back.packed_host(), t.packed_host())


def test_json_errors(tmp_path, rng):
    p = tmp_path / "bad.json"
    p.write_text("{not json")
    with pytest.raises(ValidationError, match="not valid JSON"):
        load_tensor(p)
    with pytest.raises(ValidationError, match="cannot read"):
        load_tensor(tmp_path / "missing.json")
    doc = _tensor(5, 3, 2, rng).to_doc()
    doc["blocks"][0]["j"] = [2, 1, 1]
    p.write_text(json.dumps(doc))
    with pytest.raises(ValidationError, match="not sorted"):
        load_tensor(p)
    doc = _tensor(5, 3, 2, rng).to_doc()
    doc["blocks"].pop()
    p.write_text(json.dumps(doc))
    with pytest.raises(ValidationError, match="missing block keys"):
        load_tensor(p)


@pytest.mark.parametrize("n,m,b", [(5, 3, 2), (7, 4, 3), (12, 6, 3), (4, 2, 5)])
def test_packed_roundtrip_host(n, m, b, rng, tmp_path):
    t = _tensor(n, m, b, rng)
    p = tmp_path / "t.bcg"
    save_packed(t, p)
    back = load_packed(p, device=None)
    np.testing.assert_array_equal(np.asarray(back.packed_host()), t.packed_host())
    assert back.get((1,) * m) == t.get((1,) * m)
    # the JSON and the packed codecs describe the same tensor
    emit_tensor(back, tmp_path / "t.json")
    np.testing.assert_array_equal(load_tensor(tmp_path / "t.json").packed_host(), t.packed_host())


def test_packed_errors(rng, tmp_path):
    t = _tensor(7, 4, 3, rng)
    p = tmp_path / "t.bcg"
    save_packed(t, p)
    raw = p.read_bytes()
    (tmp_path / "magic.bcg").write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(ValidationError, match="bad magic"):
        load_packed(tmp_path / "magic.bcg", device=None)
    (tmp_path / "short.bcg").write_bytes(raw[:-8])
    with pytest.raises(ValidationError, match="expected .* bytes"):
        load_packed(tmp_path / "short.bcg", device=None)
    hlen = int(np.frombuffer(raw[8:16], dtype="<u8")[0])
    hdr = json.loads(raw[16:16 + hlen].decode())
    hdr["K"] += 1
    new = json.dumps(hdr).encode()
    new += b" " * (-len(new) % 8)
    (tmp_path / "hdr.bcg").write_bytes(raw[:8] + np.uint64(len(new)).astype("<u8").tobytes() + new + raw[16 + hlen:])
    with pytest.raises(ValidationError, match="do not match"):
        load_packed(tmp_path / "hdr.bcg", device=None)
    # corrupt one block offset
    bad = bytearray(raw)
    bad[16 + hlen + 8:16 + hlen + 16] = np.int64(3).astype("<i8").tobytes()
    (tmp_path / "offs.bcg").write_bytes(bytes(bad))
    with pytest.raises(ValidationError, match="offsets"):
        load_packed(tmp_path / "offs.bcg", device=None)


@pytest.mark.gpu
def test_packed_roundtrip_device(rng, tmp_path, monkeypatch):
    """A device-resident cumulant streams to disk through the pinned chunk and
    back into HBM bit for bit (chunk shrunk so several chunks are exercised)."""
    import paper_1701_05420_b200 as bcg
    from paper_1701_05420_b200 import dataio

    monkeypatch.setattr(dataio, "CHUNK_BYTES", 4096)
    x = rng.standard_normal((2000, 11))
    cs = bcg.cumulants_upto(x, 4, b=3)
    p = tmp_path / "c4.bcg"
    save_packed(cs[4], p)
    back = load_packed(p)
    assert back._data is not None and back._data.is_cuda
    np.testing.assert_array_equal(back.data.cpu().numpy(), cs[4].packed_host())
