"""Pack the reference's own test suite for the conformance run (test infrastructure).

`python -m oracle.pack_reference_tests` (also run by __graft_entry__.build() when
/root/reference is present) writes oracle/_ref/reference_tests.tar from
/root/reference/pkg/tests.  oracle/_ref/ is git-ignored (the reference's sources
never enter this repo's history) but travels to the GPU box with the snapshot,
where tests/test_reference_suite_gpu.py unpacks it and runs it unmodified
against the `hashgraph` shim (tests/conformance/hashgraph -> this package).
"""

from __future__ import annotations

import hashlib
import io
import os
import tarfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
OUT_DIR = os.path.join(ROOT, "oracle", "_ref")
OUT = os.path.join(OUT_DIR, "reference_tests.tar")


def pack(src: str = SRC, out: str = OUT) -> str | None:
    if not os.path.isdir(src):
        return None
    os.makedirs(os.path.dirname(out), exist_ok=True)
    buf = io.BytesIO()
    digest = hashlib.sha256()
    with tarfile.open(fileobj=buf, mode="w") as tar:
        for name in sorted(os.listdir(src)):
            if not name.endswith(".py"):
                continue
            path = os.path.join(src, name)
            with open(path, "rb") as f:
                digest.update(name.encode() + b"\0" + f.read())
            tar.add(path, arcname=f"tests/{name}")
    tmp = out + ".tmp"
    with open(tmp, "wb") as f:
        f.write(buf.getvalue())
    os.replace(tmp, out)
    with open(out + ".sha256", "w") as f:
        f.write(digest.hexdigest() + "\n")
    return out


if __name__ == "__main__":
    print(pack())
