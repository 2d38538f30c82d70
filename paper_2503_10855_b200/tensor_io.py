"""Tensor JSON interchange, byte-compatible with the reference.

Format (/root/reference/pkg/src/skiff/runtime/values.py:135-168):
``{"dtype": "f32", "shape": [r, c], "data": [... row-major ...]}`` followed
by a newline.  ``load_tensor`` / ``dump_tensor`` mirror the reference's
functions of the same names, including two of its conventions:

  * a 0-d document loads as a numpy scalar of the dtype;
  * u8 data is written with dtype name "bool" -- the reference looks the name
    up by numpy dtype, bool's storage dtype is u8 and "bool" comes first in
    its table (values.py:117-123, 156-159).  "bool" loads back as u8, so the
    round trip is exact and our files are byte-identical to the reference's.
"""
from __future__ import annotations

import json

import numpy as np

# name -> numpy storage dtype, in the reference's table order (values.py:117-123)
DTYPES = {
    "bool": np.dtype(np.uint8),
    "i8": np.dtype("i1"), "i16": np.dtype("i2"), "i32": np.dtype("i4"), "i64": np.dtype("i8"),
    "u8": np.dtype("u1"), "u16": np.dtype("u2"), "u32": np.dtype("u4"), "u64": np.dtype("u8"),
    "f32": np.dtype("f4"), "f64": np.dtype("f8"),
}


class TensorFormatError(Exception):
    pass


def from_doc(doc: dict, where: str = "<doc>"):
    name = doc.get("dtype")
    if name not in DTYPES:
        raise TensorFormatError(f"unknown dtype {name!r} in {where}")
    shape = tuple(int(x) for x in doc["shape"])
    data = np.asarray(doc["data"], dtype=DTYPES[name])
    if shape == ():
        v = data.reshape(()).item()
        return v if name == "bool" else DTYPES[name].type(v)
    return data.reshape(shape)


def to_doc(value) -> dict:
    arr = value if isinstance(value, np.ndarray) else np.asarray(value)
    if arr.dtype == np.bool_:
        return {"dtype": "bool", "shape": list(arr.shape), "data": [x.item() for x in arr.astype(np.uint8).reshape(-1)]}
    for name, dt in DTYPES.items():
        if dt == arr.dtype:
            return {"dtype": name, "shape": list(arr.shape), "data": [x.item() for x in arr.reshape(-1)]}
    raise TensorFormatError(f"cannot serialize dtype {arr.dtype}")


def load_tensor(path: str):
    """Read one tensor document (values.py:135-148)."""
    with open(path) as f:
        return from_doc(json.load(f), path)


def dump_tensor(value, path: str) -> None:
    """Write one tensor document (values.py:151-168)."""
    doc = to_doc(value)
    with open(path, "w") as f:
        json.dump(doc, f)
        f.write("\n")
