"""Command line for the einsum path: ``python -m paper_2503_04771_b200.cli einsum``.

Mirrors bridgegen's ``einsum`` subcommand (cli.py:63-66, 286-322): parse the
spec, optionally check ``--shapes`` (same messages), build and print the
module (``--out`` writes it to a file).  SURVEY §8f row 3 asks for the
``--run`` extension the reference lacks (cli.py:286-299 only prints): with
``--run`` the module is executed on the B200 through ``run_function`` on
seeded random inputs of ``--shapes`` and a one-line summary is printed
(kernel(s) launched, device time, output checksum).  Only the einsum
subcommand is provided — the reference's ``gen``/``run`` front-end commands
are outside the hot path.
"""

from __future__ import annotations

import argparse
import json
import sys

from . import einsum as E


class CliError(Exception):
    """Reported on stderr with exit code 1 (bridgegen cli.py:33-34)."""


_ELEMS = {"f32": E.F32, "f64": E.F64, "bf16": E.BF16, "f16": E.F16}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="paper_2503_04771_b200",
        description="Build, print and run einsum modules on the B200 backend.")
    sub = parser.add_subparsers(dest="command", required=True)
    es = sub.add_parser("einsum", help="print (and optionally run) a module for an einsum spec")
    es.add_argument("spec", help="einsum spec, e.g. '(i,k),(k,j)->(i,j)'")
    es.add_argument("--shapes", help="comma-separated operand shapes, e.g. 4x3,3x5,4x5")
    es.add_argument("--out", help="write the printed module here instead of stdout")
    es.add_argument("--elem", default="f32", choices=sorted(_ELEMS),
                    help="element type of the module (f32/f64 as in the reference; bf16/f16)")
    es.add_argument("--schedule", help="tiling parameters, e.g. 'tile_n=512,cta_group=2'")
    es.add_argument("--run", action="store_true",
                    help="execute on the GPU with seeded random inputs of --shapes")
    es.add_argument("--seed", type=int, default=0)
    return parser


def _emit(text: str, out_path):
    if out_path:
        try:
            with open(out_path, "w", encoding="utf-8") as f:
                f.write(text)
        except OSError as e:
            raise CliError(f"cannot write {out_path}: {e}") from None
    else:
        sys.stdout.write(text)


def _shape_of(part: str) -> tuple:
    """``"4x8"`` -> ``(4, 8)``; anything else is bridgegen's 'bad shape'."""
    token = part.strip()
    dims = token.split("x")
    if any(not d.isdigit() for d in dims):
        raise CliError(f"bad shape '{token}'")
    return tuple(map(int, dims))


def check_shapes(spec: E.EinsumSpec, text: str):
    """Operand shapes from ``AxB,...`` (inputs, then the output), validated
    against the spec with the messages bridgegen's ``einsum`` subcommand
    prints (cli.py:302-322): shape syntax, operand count, rank per operand,
    one extent per index."""
    shapes = [_shape_of(part) for part in text.split(",")]
    operands = (*spec.inputs, spec.output)
    if len(shapes) != len(operands):
        raise CliError(f"{len(operands)} operand shape(s) expected, got {len(shapes)}")
    bound: dict = {}
    for shape, tup in zip(shapes, operands):
        if len(shape) != len(tup):
            raise CliError(f"shape {shape} does not match index tuple {tup}")
        for name, d in zip(tup, shape):
            first = bound.setdefault(name, d)
            if first != d:
                raise CliError(f"index '{name}' has inconsistent extents {first} and {d}")
    return shapes


def _run(module, shapes, elem, seed) -> dict:
    import numpy as np
    import torch

    from . import executor
    from . import interp as I
    if not torch.cuda.is_available():
        raise CliError("--run needs a CUDA device (there is no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())
    tdt = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16,
           "f16": torch.float16}[elem.name]
    gen = torch.Generator(device=dev).manual_seed(seed)
    vals = []
    for k, shp in enumerate(shapes):
        if k == len(shapes) - 1:
            t = torch.zeros(shp, dtype=tdt, device=dev)
        else:
            t = torch.randn(shp, generator=gen, device=dev, dtype=torch.float32).to(tdt)
        vals.append(I.TensorValue(elem, shp, t))
    executor.reset_launch_log()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    [out] = I.run_function(module, "einsum", vals, step_limit=None)
    e.record()
    torch.cuda.synchronize()
    data = out.data.double().cpu().numpy() if isinstance(out.data, torch.Tensor) else \
        np.asarray(out.data, dtype=np.float64)
    return {"out_shape": list(data.shape), "kernels": executor.launch_log(),
            "device_ms": round(s.elapsed_time(e), 4),
            "checksum": float(data.sum()), "abs_max": float(np.abs(data).max()) if data.size else 0.0}


def cmd_einsum(args) -> int:
    try:
        spec = E.parse_einsum(args.spec)
    except E.EinsumError as e:
        raise CliError(str(e)) from None
    shapes = check_shapes(spec, args.shapes) if args.shapes else None
    elem = _ELEMS[args.elem]
    try:
        module = E.build_einsum_function(None, spec, elem=elem, schedule=args.schedule)
    except (E.EinsumError, ValueError) as e:
        raise CliError(str(e)) from None
    _emit(E.print_module(module), args.out)
    if args.run:
        if shapes is None:
            raise CliError("--run needs --shapes")
        sys.stdout.write(json.dumps(_run(module, shapes, elem, args.seed)) + "\n")
    return 0


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(list(sys.argv[1:] if argv is None else argv))
        return {"einsum": cmd_einsum}[args.command](args)
    except CliError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except SystemExit as e:  # argparse usage errors carry code 2
        return e.code if isinstance(e.code, int) else 2


if __name__ == "__main__":
    sys.exit(main())
