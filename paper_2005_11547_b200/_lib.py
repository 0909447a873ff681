"""Build and load libdsk_b200.so (the sm_100a kernels behind the C ABI).

The library is compiled in-tree with nvcc (no JIT cache), so the built .so
travels with the repository snapshot to the GPU box.  There is no fallback:
if the library is missing or no CUDA device is present, every compute call
raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_PATH = os.environ.get("DSK_LIB_PATH") or os.path.join(PKG, "libdsk_b200.so")
HEADER = os.path.join(REPO, "include", "dsk_b200.h")
def _sources() -> list[str]:
    """Every CUDA source of the library (dsk_kernels.cu includes the headers)."""
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",           # no DFMA contraction: the reference rounds every op
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-fopenmp", "-shared", "-lgomp",
]

_lock = threading.Lock()
_lib = None


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    mtime = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, s) for s in _sources()] + [HEADER]
    return any(os.path.exists(d) and os.path.getmtime(d) > mtime for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: dict | None = None) -> str:
    """Compile csrc/dsk_kernels.cu into libdsk_b200.so for sm_100a.

    `out`/`defines` build a tuning variant (see profiles/sweep.py) instead.
    """
    with _lock:
        target = out or LIB_PATH
        if out is None and not force and not needs_build():
            return LIB_PATH
        tmp = target + ".tmp"
        dflags = [f"-D{k}={v}" for k, v in (defines or {}).items()]
        cmd = [_nvcc(), *NVCC_FLAGS, *dflags, "-o", tmp, os.path.join(CSRC, "dsk_kernels.cu")]
        res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
        if verbose:
            print(res.stdout + res.stderr)
        os.replace(tmp, target)
        return target


# (name, restype, argtypes)
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
SIGNATURES = [
    ("dsk_ctx_create", ctypes.c_int, [ctypes.c_int, _P, _P, _P, ctypes.POINTER(_P)]),
    ("dsk_ctx_destroy", ctypes.c_int, [_P]),
    ("dsk_ctx_device", ctypes.c_int, [_P]),
    ("dsk_minhash_density", _I64, [_I64]),
    ("dsk_launch_count", ctypes.c_uint64, []),
    ("dsk_icws_csr", ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _P, _P, _P]),
    ("dsk_bottomk_csr", ctypes.c_int,
     [_P, _P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("dsk_h2d_bytes", ctypes.c_uint64, []),
    ("dsk_minhash_csr", ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _P]),
    ("dsk_minhash_csr_ex", ctypes.c_int,
     [_P, _P, _P, _P, _I64, _I32, _I64, _P, _P, _P, _P, _P, _P]),
    ("dsk_minhash_hints", ctypes.c_int, [_P, _P, _P, _I64, _I64, ctypes.POINTER(_I64), _P]),
    ("dsk_minhash_csr_host", ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P]),
    ("dsk_lsh_csr", ctypes.c_int,
     [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P]),
    ("dsk_lsh_csr_ex", ctypes.c_int,
     [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P]),
    ("dsk_lsh_csr_host", ctypes.c_int,
     [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P]),
    ("dsk_darts_csr", ctypes.c_int,
     [_P, _P, _P, _P, _I64, _I64, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("dsk_hash64", ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P]),
    ("dsk_mix64", ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    ("dsk_pack_onebit", ctypes.c_int, [_P, _I64, _I32, _P, _P]),
    ("dsk_hash_peak", ctypes.c_int, [_P, _I32, _I64, _P, ctypes.POINTER(_I64), _P]),
    ("dsk_l1_csr", ctypes.c_int, [_P, _P, _I64, _P, _P]),
    ("dsk_dsk1_records", ctypes.c_int, [_I32, _I32, ctypes.c_uint64, _P, _I64, _P, _P]),
    ("dsk_exact_jaccard", ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P]),
    ("dsk_last_error", ctypes.c_char_p, []),
]


def load(build_if_needed: bool = True):
    """Load libdsk_b200.so (building it first when sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_needed and needs_build():
        build()
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run paper_2005_11547_b200._lib.build()")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().dsk_last_error()
        raise RuntimeError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")
