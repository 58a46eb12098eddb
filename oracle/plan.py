"""(k, g) device plan (§4.4).  TEST INFRASTRUCTURE ONLY.

"TPLA divides k devices into [g] group[s] of size k/g.  Each group holds a disjoint
slice of the latent axis of width 4d_h/g and replicates the complete set of head
parameters.  Within each group, the head axis is sharded across the k/g devices,
[so] each device processes h_q/(k/g) heads and 4d_h/g latent features."

Group-major numbering (reading R16): rank r is in latent group j = r div (k/g)
and holds head block i = r mod (k/g); all ranges are contiguous.
"""
from __future__ import annotations

import dataclasses


@dataclasses.dataclass(frozen=True)
class DevicePlan:
    rank: int
    shard: int        # latent group j
    head_block: int   # i
    head_begin: int
    head_end: int
    lat_begin: int
    lat_end: int
    row_width: int    # cache row elements: latent slice + replicated RoPE key

    @property
    def h_loc(self) -> int:
        return self.head_end - self.head_begin

    @property
    def w_lat(self) -> int:
        return self.lat_end - self.lat_begin


def make_plan(k: int, g: int, h_q: int, d_c: int, d_r: int, rank: int) -> DevicePlan:
    if k < 1 or g < 1 or k % g:
        raise ValueError("g must divide k")
    if d_c % g:
        raise ValueError("g must divide the latent width")
    per_group = k // g
    if h_q % per_group:
        raise ValueError("k/g must divide h_q")
    if not 0 <= rank < k:
        raise ValueError("rank out of range")
    j, i = divmod(rank, per_group)
    h_loc = h_q // per_group
    w_lat = d_c // g
    return DevicePlan(rank, j, i, i * h_loc, (i + 1) * h_loc, j * w_lat, (j + 1) * w_lat, w_lat + d_r)


def all_plans(k: int, g: int, h_q: int, d_c: int, d_r: int) -> list[DevicePlan]:
    return [make_plan(k, g, h_q, d_c, d_r, r) for r in range(k)]
