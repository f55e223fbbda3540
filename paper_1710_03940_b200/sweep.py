"""Scaling sweeps over subdomain counts on the GPU solve path: the ``bench``
and ``compare-deflation`` harnesses of the reference CLI
(pkg/src/deflamg/cli.py:216-289), same CSV headers and row formats
(cli.py:48-51), so sweep files from both can be diffed column by column.

    python -m paper_1710_03940_b200.sweep bench --mode weak --poisson 150 --subdomains 1,2,4,8 \\
        [--deflation constant,linear] [--config JSON|PATH] [--csv out.csv] [--device 0]
    python -m paper_1710_03940_b200.sweep compare-deflation --poisson 32 --subdomains 1,8,27

Weak mode scales the grid per axis so every subdomain keeps ``N``^3
unknowns (boxes_for(m) boxes of N^3); strong mode keeps the N^3 grid.  The
m subdomains of a sweep point run on one GPU (their AMG hierarchies merged
block-diagonally) unless the process runs under torchrun, where they are
spread over the ranks.  Problems are generated on the device
(csrc/gen_dev.cu, bit-identical to the reference's poisson3d).  Unlike the
reference (cli.py:53, 20M unknowns) the size is bounded only by device
memory.  The rest of the reference CLI (solve, print-config) is outside the
solve-phase scope of this package.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

from .config import SolverConfig
from .errors import ConfigError, DeflamgError

__all__ = ["BENCH_CSV_HEADER", "COMPARE_CSV_HEADER", "bench_sweep", "compare_deflation", "main"]

BENCH_CSV_HEADER = "subdomains,threads,setup_s,factorize_E_s,solve_s,iters,converged"
COMPARE_CSV_HEADER = "subdomains,unknowns,deflated_iters,deflated_converged,local_iters,local_converged"


def parse_counts(spec: str) -> list:
    try:
        counts = [int(p) for p in spec.split(",")]
    except ValueError:
        raise ConfigError(f"--subdomains: expected integers, got '{spec}'") from None
    if not counts or any(m < 1 for m in counts):
        raise ConfigError(f"--subdomains: counts must be positive, got '{spec}'")
    return counts


def parse_kinds(spec: str) -> list:
    kinds = spec.split(",")
    bad = [k for k in kinds if k not in ("constant", "linear")]
    if bad:
        raise ConfigError(f"--deflation: unknown kind '{bad[0]}'")
    return kinds


def load_config(source: str | None) -> SolverConfig:
    """A SolverConfig from a file path or an inline JSON object (cli.py:56-67)."""
    if source is None:
        return SolverConfig()
    text = source.strip()
    if not text.startswith("{"):
        from .errors import ParseError

        try:
            with open(source, "r", encoding="utf-8") as fh:
                text = fh.read()
        except OSError as exc:
            raise ParseError(f"{source}: cannot open: {exc}") from exc
    return SolverConfig.from_json(text)


def sweep_problem(mode: str, base: int, m: int, device: int | None):
    """The sweep point's problem (cli.py:219-226): rows, coordinates, rhs."""
    from . import problems

    if mode not in ("weak", "strong"):
        raise ConfigError(f"--mode: expected weak or strong, got '{mode}'")
    boxes = problems.boxes_for(m)
    shape = tuple(base * b for b in boxes) if mode == "weak" else (base, base, base)
    return problems.make_problem(shape, boxes, "poisson", device=device)


def _solver(prob, cfg, deflated, device):
    from .deflation import DeflatedSolver

    return DeflatedSolver(prob.matrix, prob.partition, config=cfg, coords=prob.coords, deflated=deflated,
                          device=device)


def bench_sweep(mode: str, base: int, counts, config: SolverConfig | None = None, kinds=None, threads: int = 1,
                device: int | None = 0) -> dict:
    """{kind: [row, ...]} with the rows of cli.py:236-248 (threads is echoed:
    the solve runs on the GPU, threads_per_subdomain has no effect there)."""
    cfg = config or SolverConfig()
    kinds = kinds or [cfg.get("deflation.kind")]
    out = {}
    for kind in kinds:
        rows = []
        for m in counts:
            prob = sweep_problem(mode, base, m, device)
            run_cfg = SolverConfig(json.loads(cfg.to_json()))
            run_cfg.set("deflation.kind", kind)
            s = _solver(prob, run_cfg, True, device)
            _, rep = s.solve(prob.rhs)
            rows.append((m, threads, f"{rep['setup_seconds']:.6f}", f"{rep['factorize_seconds']:.6f}",
                         f"{rep['solve_seconds']:.6f}", rep["iterations"], "true" if rep["converged"] else "false"))
        out[kind] = rows
    return out


def compare_deflation(base: int, counts, config: SolverConfig | None = None, device: int | None = 0) -> list:
    """Rows of cli.py:263-289: deflated vs plain block-AMG over a weak sweep."""
    cfg = config or SolverConfig()
    rows = []
    for m in counts:
        prob = sweep_problem("weak", base, m, device)
        _, drep = _solver(prob, cfg, True, device).solve(prob.rhs)
        _, lrep = _solver(prob, cfg, False, device).solve(prob.rhs)
        rows.append((m, prob.matrix.nrows, drep["iterations"], "true" if drep["converged"] else "false",
                     lrep["iterations"], "true" if lrep["converged"] else "false"))
    return rows


def csv_text(header: str, rows) -> str:
    return "\n".join([header] + [",".join(str(c) for c in row) for row in rows]) + "\n"


def _write(path: str | None, text: str, label: str | None = None):
    if path is None:
        if label is not None:
            sys.stdout.write(f"# deflation={label}\n")
        sys.stdout.write(text)
    else:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)


def _per_kind_path(path: str | None, kind: str, multiple: bool) -> str | None:
    if path is None or not multiple:
        return path
    root, ext = os.path.splitext(path)
    return f"{root}-{kind}{ext or '.csv'}"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1710_03940_b200.sweep")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("bench", "compare-deflation"):
        p = sub.add_parser(name)
        p.add_argument("--poisson", type=int, required=True, help="N: N^3 per subdomain (weak) or in total (strong)")
        p.add_argument("--subdomains", required=True, help="comma list of subdomain counts")
        p.add_argument("--config", default=None)
        p.add_argument("--deflation", default=None)
        p.add_argument("--threads", type=int, default=1)
        p.add_argument("--csv", default=None)
        p.add_argument("--device", type=int, default=0)
        if name == "bench":
            p.add_argument("--mode", default="weak", choices=["weak", "strong"])
    args = ap.parse_args(argv)
    try:
        cfg = load_config(args.config)
        counts = parse_counts(args.subdomains)
        if args.cmd == "bench":
            kinds = parse_kinds(args.deflation) if args.deflation else [cfg.get("deflation.kind")]
            res = bench_sweep(args.mode, args.poisson, counts, cfg, kinds, args.threads, args.device)
            for kind, rows in res.items():
                _write(_per_kind_path(args.csv, kind, len(kinds) > 1), csv_text(BENCH_CSV_HEADER, rows),
                       label=kind if len(kinds) > 1 else None)
        else:
            if args.deflation:
                (kind,) = parse_kinds(args.deflation)
                cfg.set("deflation.kind", kind)
            _write(args.csv, csv_text(COMPARE_CSV_HEADER, compare_deflation(args.poisson, counts, cfg, args.device)))
    except DeflamgError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
