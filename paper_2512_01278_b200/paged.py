"""Device paged KV pool: the HBM layout every hot-path kernel reads.

Layout:
    K, V : [layers][num_pages * page_size][kv_heads][head_dim]   (bf16 / fp32)
    table: [table_rows][pages_per_row] int32 physical page ids
A token's K row for one kv head is head_dim contiguous elements (256 B at
d=128 bf16), a token's row across heads is contiguous (2 KB at Hkv=8), and a
page of 16 tokens is 32 KB contiguous per layer, so dense verify reads stream
and sparse draft gathers move whole 16-byte-aligned rows.

Logical page accounting stays one token per page exactly as the reference
(kvpool.py:1-8); physical pages group ``page_size`` tokens.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N
from .errors import ContractError, ImpossibleRequestError


class PagedKvPool:
    def __init__(self, layers: int, kv_heads: int, head_dim: int, num_pages: int, page_size: int,
                 table_rows: int, pages_per_row: int, dtype: torch.dtype, device="cuda"):
        if page_size < 1 or page_size & (page_size - 1):
            raise ContractError("page_size must be a power of two")
        if num_pages < 1 or table_rows < 1 or pages_per_row < 1:
            raise ContractError("pool dimensions must be positive")
        self.layers, self.kv_heads, self.head_dim = layers, kv_heads, head_dim
        self.page_size = page_size
        self.page_shift = page_size.bit_length() - 1
        self.num_pages = num_pages
        self.dtype = dtype
        self.device = torch.device(device)
        slots = num_pages * page_size
        self.k = torch.zeros(layers, slots, kv_heads, head_dim, dtype=dtype, device=self.device)
        self.v = torch.zeros_like(self.k)
        self.table = torch.zeros(table_rows, pages_per_row, dtype=torch.int32, device=self.device)
        self._table_host = np.zeros((table_rows, pages_per_row), dtype=np.int32)
        self._dirty: set[int] = set()
        self._free = list(range(num_pages - 1, -1, -1))
        self._pending_free: list = []   # (event, pages): pages still read by an in-flight copy
        self._unmapped: dict[int, int] = {}  # row -> number of logical pages currently unmapped
        self._rows: dict[int, list[int]] = {}
        self._desc = None

    # -- descriptor ------------------------------------------------------------------
    def desc(self) -> N.PagedKvDesc:
        if self._desc is None:
            d = N.PagedKvDesc()
            d.k = self.k.data_ptr()
            d.v = self.v.data_ptr()
            d.layer_stride = self.k.stride(0)
            d.num_slots = self.k.shape[1]
            d.block_table = self.table.data_ptr()
            d.table_stride = self.table.stride(0)
            d.page_shift = self.page_shift
            d.kv_heads = self.kv_heads
            d.head_dim = self.head_dim
            d.dtype = N.dtype_code(self.dtype)
            self._desc = d
        return self._desc

    # -- page mapping ----------------------------------------------------------------
    @property
    def free_pages(self) -> int:
        self.reclaim()
        return len(self._free)

    def reclaim(self) -> None:
        """Return pages whose deferred-free event (an offload copy) has completed."""
        if not self._pending_free:
            return
        keep = []
        for ev, pages in self._pending_free:
            if ev.query():
                self._free.extend(pages)
            else:
                keep.append((ev, pages))
        self._pending_free = keep

    def shrink_row(self, row: int, tokens: int) -> int:
        """Return the physical pages of ``row`` past logical position ``tokens`` (KV rollback
        of whole pages, kvpool.py:315-336 free_tail); their contents are dead."""
        pages = self._rows.get(row, [])
        keep = -(-tokens // self.page_size)
        n = 0
        while len(pages) > keep:
            p = pages.pop()
            if p >= 0:
                self._free.append(p)
                n += 1
            self._table_host[row, len(pages)] = 0
        if n:
            self._dirty.add(row)
        return n

    @property
    def pages_per_row(self) -> int:
        return self.table.shape[1]

    def pages_of_row(self, row: int) -> list[int]:
        return list(self._rows.get(row, []))

    def ensure_tokens(self, row: int, tokens: int) -> None:
        """Map enough physical pages for logical positions [0, tokens) of ``row``."""
        need = -(-tokens // self.page_size)
        if need > self.pages_per_row:
            raise ImpossibleRequestError(f"row {row} needs {need} pages > {self.pages_per_row} per row")
        pages = self._rows.setdefault(row, [])
        if need - len(pages) > len(self._free):
            self.reclaim()
        if need - len(pages) > len(self._free):
            raise ImpossibleRequestError("device KV pool exhausted")
        while len(pages) < need:
            p = self._free.pop()
            self._table_host[row, len(pages)] = p
            pages.append(p)
            self._dirty.add(row)

    def release_row(self, row: int) -> None:
        for p in reversed(self._rows.pop(row, [])):
            if p >= 0:
                self._free.append(p)
        self._unmapped.pop(row, None)

    # -- host offload: physical pages leave / rejoin a row ---------------
    def unmap_pages(self, row: int, logical_pages, after=None) -> int:
        """Return the physical pages behind ``logical_pages`` of ``row`` to the free
        list (their rows were copied to the host) — once ``after`` (a CUDA event of that
        copy) has completed, when given.  The block-table entries point at page 0 until
        remapped; BatchedDecoder refuses to schedule a row with unmapped pages."""
        pages = self._rows.get(row, [])
        n = 0
        freed = []
        for lp in logical_pages:
            if lp < len(pages) and pages[lp] >= 0:
                freed.append(pages[lp])
                pages[lp] = -1
                self._table_host[row, lp] = 0
                n += 1
        if after is None:
            self._free.extend(freed)
        elif freed:
            self._pending_free.append((after, freed))
        if n:
            self._unmapped[row] = self._unmapped.get(row, 0) + n
        if n:
            self._dirty.add(row)
        return n

    def remap_pages(self, row: int, logical_pages) -> int:
        """Give unmapped ``logical_pages`` of ``row`` fresh physical pages."""
        pages = self._rows.get(row, [])
        todo = [lp for lp in logical_pages if lp < len(pages) and pages[lp] < 0]
        if len(todo) > len(self._free):
            self.reclaim()
        if len(todo) > len(self._free):
            raise ImpossibleRequestError("device KV pool exhausted while reloading")
        for lp in todo:
            pages[lp] = self._free.pop()
            self._table_host[row, lp] = pages[lp]
        if todo:
            self._dirty.add(row)
            self._unmapped[row] -= len(todo)
        return len(todo)

    def has_unmapped(self, row: int) -> bool:
        return self._unmapped.get(row, 0) > 0

    def unmapped_pages(self, row: int) -> list:
        return [i for i, p in enumerate(self._rows.get(row, [])) if p < 0]

    def sync_table(self) -> None:
        """Upload dirty block-table rows (host -> device), stream ordered and asynchronous:
        the rows are staged in pinned memory (torch's pinned allocator keeps a staging
        block alive until its copy ran), so the host never waits for the GPU here."""
        if not self._dirty:
            return
        rows = sorted(self._dirty)
        self._dirty.clear()
        if len(rows) > 8:
            self.table.copy_(torch.from_numpy(self._table_host).pin_memory(), non_blocking=True)
            return
        for r in rows:
            self.table[r].copy_(torch.from_numpy(self._table_host[r]).pin_memory(), non_blocking=True)

    # -- host-side views (tests / drop-in KvCache) -------------------------------------
    def slots(self, row: int, positions) -> torch.Tensor:
        pos = torch.as_tensor(np.asarray(positions, dtype=np.int64))
        pages = torch.as_tensor(self._table_host[row]).long()[pos >> self.page_shift]
        return (pages << self.page_shift) | (pos & (self.page_size - 1))

    def read(self, row: int, positions) -> tuple[torch.Tensor, torch.Tensor]:
        """K, V of ``positions``: (n, layers, kv_heads, head_dim)."""
        s = self.slots(row, positions).to(self.device)
        return self.k[:, s].transpose(0, 1), self.v[:, s].transpose(0, 1)

    def write(self, row: int, positions, k: torch.Tensor, v: torch.Tensor) -> None:
        """Store (n, layers, kv_heads, head_dim) rows at ``positions``."""
        s = self.slots(row, positions).to(self.device)
        self.k[:, s] = k.transpose(0, 1).to(self.device, self.dtype)
        self.v[:, s] = v.transpose(0, 1).to(self.device, self.dtype)
