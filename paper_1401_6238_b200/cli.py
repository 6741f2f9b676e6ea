"""``bench`` subcommand of the reference CLI, rebased on GPU timings
(reference cli.py:294-339, parser cli.py:397-405).

    python -m paper_1401_6238_b200 bench --order 3 --dims 32,64,128 [--reps 100]
        [--pad-pow2] [--format csv|json] [--out PATH] [--seed 0]

Same inputs (``default_rng(seed)``, complex N(0,1) h and m-1 vectors per
dimension, drawn in the reference's order), same records
``algorithm,order,dimension,median_seconds,reps`` and the same exit codes
(0 ok, 2 input error, 3 numerical degeneracy).  ``fast`` is the drop-in
``HankelTensor.tvp_partial`` (numpy in, numpy out, GPU kernels in between;
with ``--pad-pow2`` the power-of-two embedding length of
``cli._fast_product_padded``, cli.py:277-291).  ``naive`` is a dense
contraction of the explicit Hankel tensor, computed on the GPU with torch,
skipped when n^m exceeds DENSE_CAP exactly as the reference skips it; the
two must agree to 1e-10 (relative, cli.py:328-332) or the command exits 3.
The signal-processing subcommands (gen/fit1d/fit2d/svals) are outside the
product path and are not provided.
"""

from __future__ import annotations

import argparse
import csv
import json
import statistics
import sys
import time

import numpy as np
import torch

from . import batched
from ._device import require_cuda
from .hankel import DENSE_CAP, HankelTensor

EXIT_OK = 0
EXIT_INPUT = 2
EXIT_DEGENERATE = 3


class CliInputError(Exception):
    pass


class DegenerateSystemError(Exception):
    """Same role as the reference's decompose.DegenerateSystemError."""


def _parse_int_list(text):
    try:
        return [int(tok) for tok in text.split(",") if tok.strip()]
    except ValueError as exc:
        raise CliInputError(f"cannot parse integer list {text!r}: {exc}") from None


def _write_table(rows, header, fmt, out_path):
    """cli.py:135-152: JSON list of records, or CSV with a header row."""
    if fmt == "json":
        text = json.dumps([dict(zip(header, row)) for row in rows], indent=2) + "\n"
        if out_path:
            with open(out_path, "w") as fh:
                fh.write(text)
        else:
            sys.stdout.write(text)
        return
    fh = open(out_path, "w", newline="") if out_path else sys.stdout
    try:
        writer = csv.writer(fh, lineterminator="\n")
        writer.writerow(header)
        writer.writerows(rows)
    finally:
        if out_path:
            fh.close()


def _naive_product(h, shape, xs, dev):
    """Dense contraction of H[i_1..i_m] = h[i_1+..+i_m] with x_2..x_m on the
    GPU (the reference's core.dense_hankel + core.tvp_partial, cli.py:272-274)."""
    m = len(shape)
    idx = torch.zeros((), dtype=torch.int64, device=dev)
    for p, n in enumerate(shape):
        ar = torch.arange(n, device=dev).reshape([n if q == p else 1 for q in range(m)])
        idx = idx + ar
    T = torch.from_numpy(h).to(dev)[idx]
    for x in reversed(xs):
        T = T @ torch.from_numpy(x).to(dev)
    return T.cpu().numpy()


def _fast_product_padded(h, shape, xs, dev):
    """cli.py:277-291: the power-of-two embedding length."""
    dof = sum(shape) - len(shape) + 1
    length = 1
    while length < dof:
        length *= 2
    dh = torch.from_numpy(h).to(dev)[None]
    dxs = [torch.from_numpy(x).to(dev)[None] for x in xs]
    return batched.hankel_tvp_partial(dh, dxs, shape, fft_len=length)[0].cpu().numpy()


def _median_time(fn, reps):
    fn()  # warm-up
    times = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        times.append(time.perf_counter() - t0)
    return statistics.median(times), out


def cmd_bench(args) -> int:
    """cli.py:294-339."""
    if args.reps < 1:
        raise CliInputError("--reps must be at least 1")
    sizes = _parse_int_list(args.dims)
    if not sizes or any(n < 2 for n in sizes):
        raise CliInputError("--dims must list sizes of at least 2")
    m = args.order
    dev = f"cuda:{require_cuda()}"
    rng = np.random.default_rng(args.seed)
    rows = []
    for n in sizes:
        shape = (n,) * m
        dof = m * n - m + 1
        h = rng.standard_normal(dof) + 1j * rng.standard_normal(dof)
        xs = [rng.standard_normal(n) + 1j * rng.standard_normal(n) for _ in range(m - 1)]
        tensor = HankelTensor(shape, h)
        if args.pad_pow2:
            fast = lambda: _fast_product_padded(h, shape, xs, dev)  # noqa: E731
        else:
            fast = lambda: tensor.tvp_partial(xs)  # noqa: E731
        t_fast, y_fast = _median_time(fast, args.reps)
        rows.append(["fast", m, n, t_fast, args.reps])
        if n ** m > DENSE_CAP:
            rows.append(["naive", m, n, "skipped", args.reps])
            continue
        t_naive, y_naive = _median_time(lambda: _naive_product(h, shape, xs, dev), args.reps)
        err = np.linalg.norm(y_fast - y_naive) / (np.linalg.norm(y_naive) + 1.0)
        if err > 1e-10:
            raise DegenerateSystemError(f"fast and naive products disagree at n={n}: {err:.2e}")
        rows.append(["naive", m, n, t_naive, args.reps])
    _write_table(rows, ["algorithm", "order", "dimension", "median_seconds", "reps"],
                 args.format, args.out)
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    """cli.py:346-405, ``bench`` only."""
    parser = argparse.ArgumentParser(prog="hankelfft-b200")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bench", help="time naive vs fast Hankel products")
    p.add_argument("--order", type=int, default=3)
    p.add_argument("--dims", required=True, help="dimensions to sweep, e.g. '32,64,128'")
    p.add_argument("--reps", type=int, default=100)
    p.add_argument("--pad-pow2", action="store_true",
                   help="pad FFT lengths to powers of two (timing study only)")
    p.add_argument("--format", choices=["csv", "json"], default="csv")
    p.add_argument("--out", metavar="PATH", default=None)
    p.add_argument("--seed", type=int, default=0)
    p.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    """cli.py:409-425: argparse errors -> 2, input errors -> 2, degeneracy -> 3."""
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return EXIT_INPUT if exc.code not in (0, None) else 0
    try:
        return args.func(args)
    except CliInputError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INPUT
    except (DegenerateSystemError, np.linalg.LinAlgError) as exc:
        print(f"numerical degeneracy: {exc}", file=sys.stderr)
        return EXIT_DEGENERATE
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INPUT


def entrypoint():
    raise SystemExit(main())
