"""Data and tensor I/O: CSV ingestion, the reference's JSON document codec and
a packed binary format.

* ``ingest_csv`` / ``write_csv`` -- the reference's CSV contract
  (bc/dataio.py:23-86: '.' decimals, optional single header line, ragged /
  non-numeric / non-finite cells rejected with 1-based row and column), with
  a vectorised parse (numpy's C reader) and the reference's line-by-line
  parser kept for the error messages; ``device="cuda"`` lands the matrix in
  HBM through a pinned buffer (the host ingest path).

* ``emit_tensor`` / ``load_tensor`` -- the reference's JSON document
  (bc/dataio.py:89-106 over BlockSymTensor.to_doc/from_doc,
  bc/symtensor.py:219-274), same layout validation and errors.  Practical only
  for small tensors: cfg5's C6 is 2.5e9 values.
* ``save_packed`` / ``load_packed`` -- the packed buffer itself (SURVEY §8f
  row 2): a fixed header, the int64 block offsets, then the float64 values in
  the reference's packed order (sorted keys, lexicographic; row-major blocks).
  Device tensors stream to disk through one reusable pinned host chunk and
  load back the same way (never a whole-tensor host copy); the file can also
  be memory-mapped on the host (``load_packed(path, device=None)``).

File layout (little endian)::

    0   8 bytes   magic b"BCGPACK1"
    8   u64       header length H (bytes of UTF-8 JSON that follow)
    16  H bytes   {"n", "m", "b", "K", "size", "offs_sha256"} (padded with spaces to 8 B)
    ..  (K+1) i64 block offsets (the layout's ``offs``)
    ..  size f64  packed values
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from .errors import ValidationError
from .layout import layout
from .symtensor import BlockSymTensor

MAGIC = b"BCGPACK1"


def _ingest_slow(path, lines):
    """The reference's parser (bc/dataio.py:36-76), for exact diagnostics."""
    def parse_line(line):
        try:
            return [float(c) for c in line.split(",")]
        except ValueError:
            return None

    first = parse_line(lines[0])
    start = 0 if first is not None else 1
    if first is None and len(lines) == 1:
        raise ValidationError(f"{path}: no numeric rows")
    rows = []
    width = None
    for lineno, line in enumerate(lines[start:], start=1):
        cells = line.split(",")
        if width is None:
            width = len(cells)
        elif len(cells) != width:
            raise ValidationError(f"{path}: row {lineno} has {len(cells)} cells, expected {width}")
        values = []
        for col, cell in enumerate(cells, start=1):
            try:
                v = float(cell)
            except ValueError:
                raise ValidationError(
                    f"{path}: non-numeric cell at row {lineno}, column {col}: {cell.strip()!r}") from None
            if not np.isfinite(v):
                raise ValidationError(f"{path}: non-finite value at row {lineno}, column {col}")
            values.append(v)
        rows.append(values)
    if not rows:
        raise ValidationError(f"{path}: no numeric rows")
    return np.array(rows, dtype=np.float64)


def ingest_csv(path, device=None):
    """Read a t x n observation matrix from a CSV file (bc/dataio.py:23-76).

    Returns a C-contiguous float64 numpy array, or with ``device="cuda"`` a
    CUDA tensor uploaded through page-locked memory."""
    from pathlib import Path

    path = Path(path)
    try:
        text = path.read_text(encoding="utf-8")
    except OSError as exc:
        raise ValidationError(f"cannot read {path}: {exc}") from exc
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise ValidationError(f"{path}: file is empty")
    try:
        [float(c) for c in lines[0].split(",")]
        start = 0
    except ValueError:
        start = 1
    arr = None
    if len(lines) > start:
        try:
            arr = np.loadtxt(lines[start:], delimiter=",", dtype=np.float64, comments=None, ndmin=2)
        except ValueError:
            arr = None  # ragged or non-numeric: the reference parser names the cell
    if arr is None or not np.isfinite(arr).all():
        arr = _ingest_slow(path, lines)  # raises with the reference's message
    arr = np.ascontiguousarray(arr)
    if device is None:
        return arr
    from ._native import torch_cuda

    torch = torch_cuda()
    pinned = torch.from_numpy(arr).pin_memory()
    return pinned.to(device)


def write_csv(path, data, header=None) -> None:
    """Write an observation matrix as CSV with round-trip-exact floats
    (bc/dataio.py:79-86)."""
    arr = data.detach().cpu().numpy() if hasattr(data, "detach") else np.asarray(data, dtype=np.float64)
    if arr.ndim != 2:
        raise ValidationError(f"data must be 2-D, got shape {arr.shape}")
    with open(path, "w", encoding="utf-8") as fh:
        if header is not None:
            fh.write(",".join(header) + "\n")
        for row in arr:
            fh.write(",".join(repr(float(v)) for v in row) + "\n")


CHUNK_BYTES = 256 << 20  # pinned staging chunk for device tensors


def emit_tensor(tensor: BlockSymTensor, path) -> None:
    """Write a block tensor as the reference's JSON document (bc/dataio.py:89-95)."""
    doc = tensor.to_doc()
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, separators=(",", ":"))
        fh.write("\n")


def load_tensor(path) -> BlockSymTensor:
    """Read a JSON block tensor document, validating the layout (bc/dataio.py:98-106)."""
    try:
        with open(path, "r", encoding="utf-8") as fh:
            doc = json.load(fh)
    except OSError as exc:
        raise ValidationError(f"cannot read {path}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise ValidationError(f"{path}: not valid JSON: {exc}") from exc
    return BlockSymTensor.from_doc(doc)


def _offs_digest(offs: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(offs, dtype="<i8").tobytes()).hexdigest()


def save_packed(tensor: BlockSymTensor, path) -> None:
    """Write the packed buffer (header + offsets + values) to ``path``."""
    lay = layout(tensor.n, tensor.m, tensor.b)
    offs = np.asarray(lay.offs, dtype="<i8")
    hdr = json.dumps({"n": tensor.n, "m": tensor.m, "b": tensor.b, "K": int(lay.K), "size": int(lay.size),
                      "offs_sha256": _offs_digest(offs)}).encode()
    hdr += b" " * (-len(hdr) % 8)
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(np.uint64(len(hdr)).astype("<u8").tobytes())
        fh.write(hdr)
        fh.write(offs.tobytes())
        dev = tensor._data  # device buffer, if the tensor lives in HBM
        if dev is None or tensor._host is not None:
            fh.write(np.ascontiguousarray(tensor.packed_host(), dtype="<f8").tobytes())
            return
        import torch

        n = dev.numel()
        step = max(1, CHUNK_BYTES // 8)
        pinned = torch.empty(min(n, step), dtype=torch.float64, pin_memory=True)
        for lo in range(0, n, step):
            hi = min(n, lo + step)
            pinned[: hi - lo].copy_(dev[lo:hi])  # synchronous D2H into the pinned chunk
            fh.write(pinned[: hi - lo].numpy().tobytes())


def _read_header(fh, path):
    if fh.read(8) != MAGIC:
        raise ValidationError(f"{path}: not a packed tensor file (bad magic)")
    raw = fh.read(8)
    if len(raw) != 8:
        raise ValidationError(f"{path}: truncated header")
    hlen = int(np.frombuffer(raw, dtype="<u8")[0])
    if hlen > 1 << 20:
        raise ValidationError(f"{path}: implausible header length {hlen}")
    try:
        hdr = json.loads(fh.read(hlen).decode())
        n, m, b, K, size = (int(hdr[k]) for k in ("n", "m", "b", "K", "size"))
    except (ValueError, KeyError, TypeError) as exc:
        raise ValidationError(f"{path}: malformed header: {exc}") from exc
    if n < 1 or m < 1 or b < 1:
        raise ValidationError("n, m and b must all be >= 1")
    lay = layout(n, m, b)
    if K != lay.K or size != lay.size:
        raise ValidationError(f"{path}: header K={K}, size={size} do not match the (n={n}, m={m}, b={b}) layout "
                              f"(K={lay.K}, size={lay.size})")
    return n, m, b, lay, 16 + hlen, hdr


def load_packed(path, device="cuda") -> BlockSymTensor:
    """Read a packed tensor file.  ``device="cuda"``: the values go to HBM in
    pinned chunks (a device-resident tensor); ``device=None``: the values are
    memory-mapped read-only on the host."""
    with open(path, "rb") as fh:
        n, m, b, lay, pos, hdr = _read_header(fh, path)
        offs = np.frombuffer(fh.read(8 * (lay.K + 1)), dtype="<i8")
    if offs.size != lay.K + 1 or not np.array_equal(offs, np.asarray(lay.offs, dtype=np.int64)):
        raise ValidationError(f"{path}: block offsets do not match the reference layout")
    if hdr.get("offs_sha256") not in (None, _offs_digest(offs)):
        raise ValidationError(f"{path}: offsets digest mismatch")
    start = pos + 8 * (lay.K + 1)
    want = start + 8 * lay.size
    have = os.path.getsize(path)
    if have != want:
        raise ValidationError(f"{path}: expected {want} bytes, found {have}")
    vals = np.memmap(path, dtype="<f8", mode="r", offset=start, shape=(lay.size,)) if lay.size else np.empty(0)
    if device is None:
        return BlockSymTensor(n, m, b, host=vals)
    from ._native import torch_cuda

    torch = torch_cuda()
    out = torch.empty(lay.size, dtype=torch.float64, device=device)
    step = max(1, CHUNK_BYTES // 8)
    pinned = torch.empty(min(max(lay.size, 1), step), dtype=torch.float64, pin_memory=True)
    for lo in range(0, lay.size, step):
        hi = min(lay.size, lo + step)
        pinned[: hi - lo].numpy()[:] = vals[lo:hi]
        out[lo:hi].copy_(pinned[: hi - lo])  # synchronous H2D (the chunk is reused next)
    return BlockSymTensor(n, m, b, data=out)
