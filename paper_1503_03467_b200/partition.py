"""Row-strip partition of the level grids: the first building block of the
multi-GPU transform.

Every localized patch solve is independent given its level operator
(gamblet_fast.py:464-498 for the mass patches, :546-580 for the correction
patches), so a level's patches split into contiguous strips of
grid rows of the patch centres.  Rank r solves the patches of its strip with
the row-range kernels (`gb_mass_patches_rows`, `gb_correction_patches_rows`)
and writes only its rows of the output (psi^(q) windows, D^T rows), which are
contiguous in the box layout; the strips are then exchanged so every rank
holds the whole level (one broadcast per strip: strips differ by at most one
row, so this is not an equal-split all-gather).

`Strips(world)` without a process group runs every strip in this process, one
after the other on the same stream: the single-GPU check that the union of a
partition's strips is the whole-level call, bitwise.  With a process group it
is the distributed path (NCCL on GPUs, gloo on CPU tensors in the tests).
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidArgumentError


def row_strips(L, world):
    """Balanced contiguous row ranges [(r0, r1)] covering [0, L): the first
    L % world ranks get one row more."""
    L, world = int(L), int(world)
    if world < 1:
        raise InvalidArgumentError(f"world must be >= 1, got {world}")
    if L < 0:
        raise InvalidArgumentError(f"L must be >= 0, got {L}")
    base, extra = divmod(L, world)
    out, r0 = [], 0
    for r in range(world):
        r1 = r0 + base + (1 if r < extra else 0)
        out.append((r0, r1))
        r0 = r1
    return out


@dataclass
class Strips:
    """A row-strip partition: `world` strips, this process owns `rank`'s;
    group None with distributed=False runs all strips in-process."""
    world: int
    rank: int = 0
    distributed: bool = False
    group: object = None

    def owned(self, L):
        return [row_strips(L, self.world)[self.rank]] if self.distributed else \
            row_strips(L, self.world)


def gather_strips(buf, L, row_elems, strips):
    """Complete `buf` (row-major, `row_elems` elements per grid row) on every
    rank after each rank wrote the rows of its own strip."""
    if not strips.distributed or strips.world == 1:
        return
    import torch.distributed as dist
    for r, (a, b) in enumerate(row_strips(L, strips.world)):
        if b > a:
            dist.broadcast(buf[a * row_elems:b * row_elems], src=r, group=strips.group)


def run_strips(strips, L, row_elems, buf, solve):
    """solve(r0, r1) for the owned strips, then the exchange."""
    for r0, r1 in strips.owned(L):
        if r1 > r0:
            solve(r0, r1)
    gather_strips(buf, L, row_elems, strips)
