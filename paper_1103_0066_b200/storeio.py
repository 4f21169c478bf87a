"""The reference's on-disk formats from Python:

* FBEMAT01 element-matrix store (reference src/engine.cpp:413-508): magic
  "FBEMAT01", u32 dim, krows, element_batch_size, num_concurrent_elements,
  u64 num_elements, u32 precision (0 f32, 1 f64), then the store scalars;
  little-endian.
* text mesh (reference src/geometry.cpp:353-395): "dim nv ne", one vertex per
  line, then one cell per line, doubles at 17 significant digits.

Byte-exact with files the unmodified reference wrote (tests/golden/*.fbemat,
*.mesh; tests/test_storeio.py).  Host-side file formats: numpy in, numpy out.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

MAGIC = b"FBEMAT01"
_HDR = struct.Struct("<IIIIQI")


@dataclass
class StoreFile:
    dim: int
    krows: int
    element_batch_size: int
    num_concurrent_elements: int
    num_elements: int
    data: np.ndarray  # float32 / float64, num_batches * bs * krows^2 scalars


def write_store(path: str, data, dim: int, krows: int, element_batch_size: int, num_elements: int,
                num_concurrent_elements: int = 1) -> None:
    a = data.cpu().numpy() if type(data).__module__.startswith("torch") else np.asarray(data)
    if a.dtype not in (np.float32, np.float64):
        raise ValueError("store scalars must be float32 or float64")
    nb = -(-num_elements // element_batch_size)
    if a.size != nb * element_batch_size * krows * krows:
        raise ValueError("store length does not match num_batches * bs * krows^2")
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(_HDR.pack(dim, krows, element_batch_size, num_concurrent_elements, num_elements,
                          0 if a.dtype == np.float32 else 1))
        f.write(np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<"), copy=False).tobytes())


def read_store(path: str) -> StoreFile:
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ValueError("not an element-matrix store file")
        hdr = f.read(_HDR.size)
        if len(hdr) != _HDR.size:
            raise ValueError("truncated element-matrix store header")
        dim, kr, bs, ce, ne, pc = _HDR.unpack(hdr)
        if dim not in (2, 3) or kr <= 0 or bs <= 0 or ce <= 0 or bs % ce or pc > 1:
            raise ValueError("store header: bad shape or precision code")
        dt = np.dtype("<f4" if pc == 0 else "<f8")
        n = -(-ne // bs) * bs * kr * kr
        raw = f.read(n * dt.itemsize)
        if len(raw) != n * dt.itemsize:
            raise ValueError("truncated element-matrix store data")
        return StoreFile(dim, kr, bs, ce, ne, np.frombuffer(raw, dtype=dt).astype(dt.newbyteorder("=")))


def write_mesh_text(path: str, vertices, cells, dim: int) -> None:
    v = np.asarray(vertices, dtype=np.float64).reshape(-1, dim)
    c = np.asarray(cells, dtype=np.int32).reshape(-1, dim + 1)
    lines = [f"{dim} {v.shape[0]} {c.shape[0]}"]
    lines += [" ".join(_g17(x) for x in row) for row in v]
    lines += [" ".join(str(int(x)) for x in row) for row in c]
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def read_mesh_text(path: str):
    with open(path) as f:
        tok = f.read().split()
    dim, nv, ne = int(tok[0]), int(tok[1]), int(tok[2])
    v = np.array(tok[3:3 + nv * dim], dtype=np.float64)
    c = np.array(tok[3 + nv * dim:3 + nv * dim + ne * (dim + 1)], dtype=np.int32)
    if v.size != nv * dim or c.size != ne * (dim + 1):
        raise ValueError("truncated mesh file")
    return dim, v, c


def _g17(x: float) -> str:
    return "%.17g" % x


# ---------------------------------------------------------------- bench records
# The reference's benchmark table (src/bench.cpp:231-384; the C++ layer's
# write_csv / read_csv / write_json): 15 fields, string fields quoted with
# doubled quotes, flags "on"/"off", doubles at 17 significant digits.
CSV_HEADER = ("operator,dim,num_elements,batch_size,concurrent,interleave,unroll,"
              "precision,workers,reps,seconds_min,seconds_mean,gflops,checksum,status")
_FIELDS = CSV_HEADER.split(",")
_INT = {"dim", "num_elements", "batch_size", "concurrent", "workers", "reps"}
_FLT = {"seconds_min", "seconds_mean", "gflops", "checksum"}
_FLAG = {"interleave", "unroll"}


def _q(s: str) -> str:
    return '"' + s.replace('"', '""') + '"'


def write_bench_csv(path: str, records, extra=()) -> None:
    """records: dicts keyed by the CSV field names (flags as bools).  `extra`
    names extension columns appended after the reference's 15 (numbers at 17
    significant digits, None as an empty cell); with none the file is the
    reference's format byte for byte."""
    with open(path, "w", newline="") as f:
        f.write(CSV_HEADER + "".join("," + k for k in extra) + "\n")
        for r in records:
            out = []
            for k in _FIELDS:
                v = r[k]
                if k in _FLAG:
                    out.append(_q("on" if v else "off"))
                elif k in _FLT:
                    out.append(_g17(float(v)))
                elif k in _INT:
                    out.append(str(int(v)))
                else:
                    out.append(_q(str(v)))
            for k in extra:
                v = r.get(k)
                out.append("" if v is None else (str(v) if isinstance(v, int) else _g17(float(v))))
            f.write(",".join(out) + "\n")


def _split(line: str):
    fields, cur, q, i = [], "", False, 0
    while i < len(line):
        ch = line[i]
        if q:
            if ch == '"':
                if i + 1 < len(line) and line[i + 1] == '"':
                    cur += '"'
                    i += 1
                else:
                    q = False
            else:
                cur += ch
        elif ch == '"':
            q = True
        elif ch == ",":
            fields.append(cur)
            cur = ""
        else:
            cur += ch
        i += 1
    fields.append(cur)
    return fields


def read_bench_csv(path: str):
    """Records as dicts; the reference reader's errors (ValueError here)."""
    with open(path, newline="") as f:
        lines = f.read().split("\n")
    if not lines or lines == [""]:
        raise ValueError("empty benchmark table")
    if lines[0].rstrip("\r") != CSV_HEADER:
        raise ValueError("unrecognized benchmark table header")
    out = []
    for line in lines[1:]:
        line = line.rstrip("\r")
        if not line:
            continue
        f = _split(line)
        if len(f) != 15:
            raise ValueError(f"benchmark table row has {len(f)} fields, expected 15")
        r = {}
        for k, v in zip(_FIELDS, f):
            if k in _FLAG:
                if v not in ("on", "off"):
                    raise ValueError(f"bad flag field '{v}' (want on/off)")
                r[k] = v == "on"
            elif k in _INT:
                r[k] = int(v)
            elif k in _FLT:
                r[k] = float(v)
            else:
                r[k] = v
        out.append(r)
    return out


def write_bench_json(path: str, records) -> None:
    """Array of objects in CSV field order, flags as "on"/"off"."""
    import json
    rows = [{k: (("on" if r[k] else "off") if k in _FLAG else r[k]) for k in _FIELDS} for r in records]
    with open(path, "w") as f:
        f.write(json.dumps(rows, indent=2) + "\n")
