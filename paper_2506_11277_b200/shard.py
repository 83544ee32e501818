"""2-D C-tile sharding of the Ozaki-I GEMM over the ranks of one node.

C is split into p_r x p_c blocks (1x1, 2x1, 2x2, 4x2 for 1/2/4/8 ranks,
SURVEY.md section 8e).  Rank r owns block (i, j) = divmod(r, p_c) and needs A
row-panel i and B column-panel j with the full inner dimension.  Scales are
per full row of A / column of B, so a block never needs another block's data
and the blocked result is bit-identical to the monolithic one (the reference's
multiply() on row/column blocks).  The only exchange step is
distributing the panels from their owners: A panel i lives on rank (i, 0),
B panel j on rank (0, j); each is broadcast along its row / column group.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple


def grid_for(world: int) -> Tuple[int, int]:
    """(p_r, p_c) with p_r >= p_c and p_r * p_c == world, as square as possible."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    best = (world, 1)
    for pc in range(1, world + 1):
        if world % pc == 0:
            pr = world // pc
            if pr >= pc:
                best = (pr, pc)
    return best


@dataclass(frozen=True)
class Block:
    rank: int
    i: int  # block row (A row-panel index)
    j: int  # block column (B column-panel index)
    row0: int
    row1: int
    col0: int
    col1: int


def split_range(n: int, parts: int, idx: int) -> Tuple[int, int]:
    base, rem = divmod(n, parts)
    lo = idx * base + min(idx, rem)
    return lo, lo + base + (1 if idx < rem else 0)


def block_of(rank: int, world: int, m: int, n: int) -> Block:
    pr, pc = grid_for(world)
    i, j = divmod(rank, pc)
    r0, r1 = split_range(m, pr, i)
    c0, c1 = split_range(n, pc, j)
    return Block(rank, i, j, r0, r1, c0, c1)


def row_group(world: int, i: int) -> List[int]:
    """Ranks sharing A row-panel i (its owner, rank (i, 0), comes first)."""
    _, pc = grid_for(world)
    return [i * pc + j for j in range(pc)]


def col_group(world: int, j: int) -> List[int]:
    """Ranks sharing B column-panel j (its owner, rank (0, j), comes first)."""
    pr, pc = grid_for(world)
    return [i * pc + j for i in range(pr)]


def a_owner(world: int, i: int) -> int:
    return row_group(world, i)[0]


def b_owner(world: int, j: int) -> int:
    return col_group(world, j)[0]


class PanelExchange:
    """The exchange step of a sharded multiply, shared by bench.py (NCCL, CUDA
    tensors) and the gloo tests (CPU tensors): one process group per block row
    and per block column, created collectively in the same order on every
    rank; `exchange` broadcasts A row-panel i from rank (i, 0) along row
    group i and B column-panel j from rank (0, j) along column group j."""

    def __init__(self, world: int, rank: int):
        import torch.distributed as dist
        self.world, self.rank = world, rank
        self.pr, self.pc = grid_for(world)
        self.i, self.j = divmod(rank, self.pc)
        self.row_groups = [dist.new_group(row_group(world, i)) for i in range(self.pr)] \
            if world > 1 else []
        self.col_groups = [dist.new_group(col_group(world, j)) for j in range(self.pc)] \
            if world > 1 else []

    def exchange(self, a_panel, b_panel) -> None:
        """In place: a_panel / b_panel hold the owner's data afterwards."""
        import torch.distributed as dist
        if self.world == 1:
            return
        if self.pc > 1:
            dist.broadcast(a_panel, src=a_owner(self.world, self.i), group=self.row_groups[self.i])
        if self.pr > 1:
            dist.broadcast(b_panel, src=b_owner(self.world, self.j), group=self.col_groups[self.j])
