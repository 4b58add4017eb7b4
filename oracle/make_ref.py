"""Copy recipe for the unmodified reference package (test / baseline
infrastructure only).

Zips /root/reference/pkg/src/zcgraph (pure Python + numpy)
into oracle/_ref/zcgraph_ref.zip, which is git-ignored but travels to the GPU
box with the repo snapshot (where /root/reference does not exist).  Python
imports packages straight from a zip (zipimport), so the reference runs there
byte-for-byte as shipped.  Only tests/ and bench.py's reference / CPU-baseline
legs import it, through oracle.reference().
"""
from __future__ import annotations

import hashlib
import os
import sys
import zipfile

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg/src/zcgraph"
OUT_DIR = os.path.join(HERE, "_ref")
ZIP = os.path.join(OUT_DIR, "zcgraph_ref.zip")


def build(force: bool = False) -> str | None:
    """(Re)build the zip when the reference tree is present; return its path
    (None when neither the tree nor a previous zip exists)."""
    if not os.path.isdir(SRC):
        return ZIP if os.path.exists(ZIP) else None
    files = sorted(f for f in os.listdir(SRC) if f.endswith(".py"))
    if not force and os.path.exists(ZIP):
        return ZIP
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = ZIP + ".tmp"
    with zipfile.ZipFile(tmp, "w", zipfile.ZIP_DEFLATED) as z:
        for f in files:  # fixed timestamp: the tree's mtimes predate 1980
            info = zipfile.ZipInfo(f"zcgraph/{f}", date_time=(2020, 6, 12, 0, 0, 0))
            info.compress_type = zipfile.ZIP_DEFLATED
            with open(os.path.join(SRC, f), "rb") as fh:
                z.writestr(info, fh.read())
    os.replace(tmp, ZIP)
    return ZIP


def digest(path: str = ZIP) -> str:
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()[:16]


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
