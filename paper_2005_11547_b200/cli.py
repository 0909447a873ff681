"""`sketch` command: a set file -> a DSK1 record stream, on the GPU.

    python -m paper_2005_11547_b200.cli sketch --input SETS.txt --out OUT.dsk \
        [--algo dartminhash|icws|icws-fast|bottomk] [--k 256] [--seed 1] [--one-bit]

The reference's `dartsketch sketch` (ref/cli.py:107-131) reads every set of
the file, then sketches them one at a time and concatenates `dump_sketch`
records.  This driver reads the file into one CSR batch (io.read_csr), runs
the batch kernel for the algorithm once over all rows, and writes the
records with the DSK1 record kernel (dsk_dsk1_records) -- byte-identical to
the reference's output file.

Errors follow the reference: a ValidationError prints `error: <message>` to
stderr and exits 2; sketch errors name the first failing set in file order,
after the whole file has been parsed (as read_sets runs before any sketch);
`--one-bit` with bottom-k fails on the first set, after that set is sketched.
Only `sketch` is provided (the estimate / timing / lsh-demo commands are
experiment harnesses outside the sketching path).
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from .constants import ValidationError

ALGORITHMS = ("dartminhash", "icws", "icws-fast", "bottomk")  # ref/bench.py:31


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="paper_2005_11547_b200.cli",
        description="GPU batch sketching of weighted-set files into DSK1 records")
    sub = parser.add_subparsers(dest="command", required=True)
    sk = sub.add_parser("sketch", help="sketch sets from a text file into a binary record stream")
    sk.add_argument("--input", required=True, help="text file, one set per line (id:weight tokens)")
    sk.add_argument("--algo", default="dartminhash", choices=ALGORITHMS)
    sk.add_argument("--k", type=int, default=256)
    sk.add_argument("--seed", type=int, default=1)
    sk.add_argument("--one-bit", action="store_true", help="emit one-bit sketches")
    sk.add_argument("--out", required=True, help="output file (binary)")
    sk.add_argument("--device", default=None, help="CUDA device (default: current)")
    return parser


def sketch_records(indptr, ids, weights, algo: str, k: int, seed: int, one_bit: bool,
                   device=None) -> bytes:
    """The DSK1 stream for every row of a CSR batch, as the reference's
    `sketch` command would write it for the same sets."""
    import torch

    from . import api
    from .api import (KIND_BOTTOMK, KIND_MINHASH, KIND_ONEBIT, HashFamily, _csr_to_dev,
                      _device, dump_sketches)

    n = int(np.asarray(indptr).size - 1)
    if n == 0:
        return b""
    indptr = np.asarray(indptr, dtype=np.int64)
    if k < 1:
        # the first set fails: IcwsSketcher(k) is built before anything else;
        # dart_minhash / bottom_k check emptiness first (ref/sketching.py:86-90)
        if algo not in ("icws", "icws-fast") and indptr[1] == indptr[0]:
            raise ValidationError("cannot sketch an empty set")
        raise ValidationError(f"k must be positive, got {k}")
    dev = _device(device)
    hashes = HashFamily(seed)
    p, i, w = _csr_to_dev(indptr, ids, weights, dev)
    if algo == "dartminhash":
        res = api.minhash_batch(p, i, w, k, hashes, values=not one_bit, bits=one_bit,
                                stats=False, device=dev, check=False)
        _raise_first(res.status)
        if (res.status != 0).any():  # DSK_STATUS_TIE rows: repair by index tuple
            api._resolve_minhash_ties(res, p, i, w, k, hashes, dev)
        if one_bit:
            return dump_sketches(res.bits, KIND_ONEBIT, k, seed)
        return dump_sketches(res.values, KIND_MINHASH, k, seed)
    if algo in ("icws", "icws-fast"):
        res = api.icws_batch(p, i, w, k, hashes, device=dev, check=False)
        _raise_first(res.status)
        # icws_fingerprints (ref/baselines.py:152-161): hash64(element,
        # w = tick & 0xffffffff, r = tick >> 32, stream 11), on the device
        el = api.as_u64(res.element).reshape(-1)
        tk = api.as_u64(res.tick).reshape(-1)
        fps = hashes.hash64_array(el, w=tk & np.uint64(0xFFFFFFFF), r=tk >> np.uint64(32),
                                  stream=11, device=dev)
        vals = torch.from_numpy(np.ascontiguousarray(fps).view(np.int64)).to(dev).reshape(n, k)
        if one_bit:
            from . import _lib
            packed = torch.empty((n, (k + 63) // 64), dtype=torch.int64, device=dev)
            with torch.cuda.device(dev):
                _lib.check(_lib.load().dsk_pack_onebit(api._ptr(vals), n, k, api._ptr(packed),
                                                       api._stream_ptr(dev)), "dsk_pack_onebit")
            return dump_sketches(packed, KIND_ONEBIT, k, seed)
        return dump_sketches(vals, KIND_MINHASH, k, seed)
    # bottom-k: the reference sketches set 0, then rejects --one-bit
    if one_bit:
        m = int(indptr[1] - indptr[0])
        first = api.bottom_k_batch(p[:2] - p[0], i[:m], w[:m], k, hashes, device=dev,
                                   check=False)
        _raise_first(first.status)
        raise ValidationError("--one-bit requires a minhash-style sketch")
    res = api.bottom_k_batch(p, i, w, k, hashes, device=dev, check=False)
    _raise_first(res.status)
    return dump_sketches(res.columns["fingerprint"], KIND_BOTTOMK, k, seed)


def _raise_first(status) -> None:
    """The reference's exception (same type and message) for the first
    failing set in file order."""
    from .api import _STATUS_ERRORS
    st = status.cpu().numpy() & 0xFF
    bad = np.nonzero(st)[0]
    if bad.size:
        exc, msg = _STATUS_ERRORS.get(int(st[bad[0]]), (RuntimeError, f"status {st[bad[0]]}"))
        raise exc(msg)


def _cmd_sketch(args) -> int:
    from .io import read_csr
    if args.out == "-":
        raise ValidationError("sketch output is binary; --out must be a file path")
    indptr, ids, weights = read_csr(args.input)
    data = sketch_records(indptr, ids, weights, args.algo, args.k, args.seed, args.one_bit,
                          args.device)
    try:
        with open(args.out, "wb") as handle:
            handle.write(data)
    except OSError as exc:
        raise ValidationError(f"cannot write {args.out!r}: {exc}") from exc
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return {"sketch": _cmd_sketch}[args.command](args)
    except ValidationError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
