"""Transform-style tiling parameters for a ``linalg.generic``.

The reference has no schedule language (the paper's transform dialect /
Halide-style scheduling is out of its scope); its generic op only
carries indexing maps and iterator types (einsum.py:85-94).  A ``Schedule``
is the B200 backend's equivalent of ``transform.structured.tile_using_forall``
parameters: it pins the kernel variant the planner would otherwise choose —
CTA group (1 CTA or a CTA pair), N tile width, pipeline depth, rasterisation,
split-K — and can be attached to a generic op:

  * mirror API: ``build_generic(ctx, registry, spec, operands, schedule=...)``
    or ``build_einsum_function(..., schedule=...)``; printed as the attribute
    ``bgx.schedule = "..."``;
  * real bridgegen IR: an extra ``StringAttr`` named ``"bgx.schedule"`` on the
    op (bridgegen's verifier checks only declared attributes,
    dialects.py:284-292), read by ``compat``.
All fields default to 0 = let the planner choose.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

_KEYS = ("tile_n", "stages", "cta_group", "raster", "splits", "max_ctas", "cluster_n")


@dataclass(frozen=True)
class Schedule:
    tile_n: int = 0       # tcgen05 N tile: 64/128/256, 512 with cta_group=2
    stages: int = 0       # smem pipeline depth
    cta_group: int = 0    # 1 = one CTA (128-row tiles), 2 = CTA pair (256-row tiles)
    raster: int = 0       # >0: groups of M tiles; <0: groups of N tiles
    splits: int = 0       # split-K slices (>1), or tail split of the last wave (<-1)
    max_ctas: int = 0     # cap on persistent CTAs
    cluster_n: int = 0    # 2: two CTA pairs per cluster along N share A by TMA multicast

    def to_dict(self) -> dict:
        return {k: v for k, v in asdict(self).items() if v}

    def __str__(self) -> str:
        return ",".join(f"{k}={v}" for k, v in asdict(self).items() if v)

    @classmethod
    def parse(cls, text: str) -> "Schedule":
        """``"tile_n=512,cta_group=2"`` → Schedule (unknown keys rejected)."""
        vals = {}
        for part in (p.strip() for p in str(text).split(",")):
            if not part:
                continue
            key, _, val = part.partition("=")
            key = key.strip()
            if key not in _KEYS:
                raise ValueError(f"unknown schedule parameter '{key}'")
            vals[key] = int(val)
        return cls(**vals)


def as_schedule_dict(schedule) -> dict | None:
    """Accept a Schedule, a dict, a string, or None."""
    if schedule is None:
        return None
    if isinstance(schedule, Schedule):
        return schedule.to_dict() or None
    if isinstance(schedule, str):
        return Schedule.parse(schedule).to_dict() or None
    return dict(schedule) or None


__all__ = ["Schedule", "as_schedule_dict"]
