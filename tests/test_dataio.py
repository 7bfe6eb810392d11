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


def test_csv_roundtrip_exact_with_header(rng, tmp_path):
    from paper_1701_05420_b200.dataio import ingest_csv, write_csv

    x = rng.standard_normal((37, 5)) * 10.0 ** rng.integers(-5, 5, (37, 5))
    write_csv(tmp_path / "a.csv", x, header=["v1", "v2", "v3", "v4", "v5"])
    np.testing.assert_array_equal(ingest_csv(tmp_path / "a.csv"), x)
    write_csv(tmp_path / "b.csv", x)
    np.testing.assert_array_equal(ingest_csv(tmp_path / "b.csv"), x)


@pytest.mark.parametrize("text,match", [
    ("1,2\n3\n", "row 2 has 1 cells, expected 2"),
    ("a,b\n1,2\n3,x\n", "non-numeric cell at row 2, column 2: 'x'"),
    ("1,2\n3,nan\n", "non-finite value at row 2, column 2"),
    ("1,inf\n", "non-finite value at row 1, column 2"),
    ("a,b\n", "no numeric rows"),
    ("\n\n", "file is empty"),
])
def test_csv_errors_match_reference_messages(text, match, tmp_path):
    """bc/dataio.py:36-76 diagnostics (1-based rows, header excluded)."""
    from paper_1701_05420_b200.dataio import ingest_csv

    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(ValidationError, match=match):
        ingest_csv(p)


def test_csv_blank_lines_and_spaces(tmp_path):
    from paper_1701_05420_b200.dataio import ingest_csv

    p = tmp_path / "s.csv"
    p.write_text("x,y\n\n 1.5, 2\n3,4e-3\n\n")
    np.testing.assert_array_equal(ingest_csv(p), np.array([[1.5, 2.0], [3.0, 4e-3]]))


@pytest.mark.gpu
def test_csv_ingest_to_device_then_cumulants(rng, tmp_path):
    """CSV -> pinned -> HBM ingest path feeding cumulants_upto (same result as
    from the in-memory array)."""
    import paper_1701_05420_b200 as bcg
    from paper_1701_05420_b200.dataio import ingest_csv, write_csv

    x = rng.exponential(1.0, (500, 4))
    write_csv(tmp_path / "x.csv", x, header=["a", "b", "c", "d"])
    X = ingest_csv(tmp_path / "x.csv", device="cuda")
    assert X.is_cuda and X.shape == (500, 4)
    a, b = bcg.cumulants_upto(X, 4, b=2), bcg.cumulants_upto(x, 4, b=2)
    for k in range(2, 5):
        np.testing.assert_array_equal(a[k].packed_host(), b[k].packed_host())
