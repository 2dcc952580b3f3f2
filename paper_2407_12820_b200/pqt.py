""".pqt files: the reference's tensor and PQ-index format (tensor.cpp:46-150,
pq.cpp:184-222), header as the code writes it (not the README's prose):

    "PQKV" | u32 version (1) | u8 dtype (0 f32, 1 u16) | u8 ndim | u64 dims[ndim]
    | little-endian payload

An index file is the centroid tensor [m][2^b][d_m] f32 followed by the code
grid [s][m] u16.  Host-side numpy I/O; `to_device` moves a loaded index into
the device layout the kernels use."""
import struct

import numpy as np

MAGIC = b"PQKV"
VERSION = 1
F32, U16 = 0, 1


def _write(f, dtype_code, arr):
    if arr.ndim < 1 or arr.ndim > 255:
        raise ValueError("tensor: ndim must be in [1, 255]")
    if any(d == 0 for d in arr.shape):
        raise ValueError("tensor: zero-sized dimension")
    f.write(MAGIC + struct.pack("<IBB", VERSION, dtype_code, arr.ndim))
    f.write(struct.pack(f"<{arr.ndim}Q", *arr.shape))
    f.write(np.ascontiguousarray(arr).astype("<f4" if dtype_code == F32 else "<u2", copy=False).tobytes())


def _read(f, want):
    head = f.read(10)
    if len(head) < 4 or head[:4] != MAGIC:
        raise RuntimeError("tensor: bad magic")
    if len(head) < 10:
        raise RuntimeError("tensor: truncated file")
    version, dtype_code, ndim = struct.unpack("<IBB", head[4:])
    if version != VERSION:
        raise RuntimeError("tensor: unsupported format version")
    if dtype_code != want:
        raise RuntimeError("tensor: unexpected dtype")
    if ndim == 0:
        raise RuntimeError("tensor: ndim must be >= 1")
    raw = f.read(8 * ndim)
    if len(raw) < 8 * ndim:
        raise RuntimeError("tensor: truncated file")
    dims = struct.unpack(f"<{ndim}Q", raw)
    if any(d == 0 for d in dims):
        raise ValueError("tensor: zero-sized dimension")
    n = int(np.prod(dims, dtype=np.uint64))
    dt = np.dtype("<f4") if want == F32 else np.dtype("<u2")
    payload = f.read(n * dt.itemsize)
    if len(payload) < n * dt.itemsize:
        raise RuntimeError("tensor: truncated payload")
    return np.frombuffer(payload, dt).reshape(dims).copy()


def write_tensor(f, t):
    t = np.asarray(t, np.float32)
    if not np.all(np.isfinite(t)):
        raise ValueError("tensor: non-finite value")
    _write(f, F32, t)


def read_tensor(f):
    t = _read(f, F32)
    if not np.all(np.isfinite(t)):
        raise ValueError("tensor: non-finite value")
    return t


def save_tensor(path, t):
    with open(path, "wb") as f:
        write_tensor(f, t)


def load_tensor(path):
    with open(path, "rb") as f:
        return read_tensor(f)


def write_index(f, centroids, codes):
    """centroids [m][2^b][d_m] f32, codes [s][m] u16 (pq.cpp:184-188)."""
    centroids = np.asarray(centroids, np.float32)
    codes = np.asarray(codes)
    m, c, _ = centroids.shape
    if c & (c - 1) or not 2 <= c <= 65536:
        raise ValueError("pq: n_clusters must be 2^b, b in [1, 16]")
    if codes.ndim != 2 or codes.shape[1] != m:
        raise ValueError("pq: code grid shape mismatch")
    write_tensor(f, centroids)
    _write(f, U16, codes.astype(np.uint16))


def read_index(f):
    """-> (centroids [m][2^b][d_m], codes [s][m] u16), validated as pq.cpp:190-213."""
    cen = read_tensor(f)
    if cen.ndim != 3:
        raise RuntimeError("pq: centroid tensor must be 3-d")
    m, c, _ = cen.shape
    if c & (c - 1) or not 2 <= c <= 65536:
        raise ValueError("pq: n_clusters must be 2^b, b in [1, 16]")
    codes = _read(f, U16)
    if codes.ndim != 2 or codes.shape[1] != m:
        raise RuntimeError("pq: code grid shape mismatch")
    if codes.size and int(codes.max()) >= c:
        raise RuntimeError("pq: code entry out of range")
    return cen, codes


def save_index(path, centroids, codes):
    with open(path, "wb") as f:
        write_index(f, centroids, codes)


def load_index(path):
    with open(path, "rb") as f:
        return read_index(f)


def to_device(centroids, codes, device="cuda"):
    """Index arrays -> the device layout of Context.pq_build: centroids [1][m][C][d_m]
    f32 and codes [1][s][m] int16 (u16 bit patterns)."""
    import torch

    cen = torch.from_numpy(np.ascontiguousarray(centroids, np.float32))[None].to(device)
    cd = torch.from_numpy(np.ascontiguousarray(codes, np.uint16).view(np.int16))[None].to(device)
    return cen, cd
