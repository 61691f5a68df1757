"""Build libb200k.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libb200k.so")
SOURCES = ["capi.cu", "transpose.cu", "transpose_tma.cu", "transpose_any.cu", "transpose_staged.cu", "transpose_cpa.cu", "reduce.cu"]
HEADERS = ["b2_internal.cuh", os.path.join("..", "..", "include", "b2k.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-Xptxas", "-v",
    "-cudart", "static",
    "-shared",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def source_id() -> str:
    """sha256 prefix of everything the library is compiled from (sources, headers,
    flags): embedded as b2_build_id() so a stale prebuilt .so is detected by
    content, not by mtime (a snapshot or copy may reset mtimes)."""
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(name.encode() + b"\0" + f.read() + b"\0")
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()[:16]


def lib_is_current(path: str = LIB) -> bool:
    """True if the .so at `path` embeds the current source_id (its b2_build_id
    string literal); checked on the file bytes, before anything is loaded."""
    if not os.path.exists(path):
        return False
    tag = b"b2k-build-" + source_id().encode()
    with open(path, "rb") as f:
        return tag in f.read()


def _stale() -> bool:
    return not lib_is_current(LIB)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    bid = "b2k-build-" + source_id()
    cmd = [nvcc(), *NVCC_FLAGS, f'-DB2_BUILD_ID="{bid}"', "-o", LIB + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write(r.stderr)
    if verbose:
        print(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
