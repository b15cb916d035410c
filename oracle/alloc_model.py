"""ORACLE (test infrastructure only) — reference model of the paged KV allocator.

Only tests/ may import it.  It replays apex_kv_alloc / apex_kv_release
sequences and predicts, bit-for-bit, the block tables, lengths and slot
mapping the library must produce.

PAPER.md never specifies paging (P:371-374 name "Paged Attention" kernels; P:156
says KV management "is handled dynamically"; P:51 one K and one V vector per
token per layer).  The allocation contract is DESIGN.md reading c10 (SURVEY.md
§8(c) c10):
  * LIFO free list, initialised so the first pop returns block 0;
  * a block is taken only when a token lands at pos % block_size == 0;
  * an alloc call is all-or-nothing (SPEC.md S:139 per-request rejection);
  * release pushes the sequence's blocks back in reverse table order, so the
    next pops return them in table order.
"""
from __future__ import annotations


class AllocError(Exception):
    def __init__(self, code: str):
        super().__init__(code)
        self.code = code          # "EINVAL" | "ENOBLOCKS" | "ESEQ"


class AllocModel:
    def __init__(self, num_blocks: int, max_seqs: int, max_blocks_per_seq: int,
                 block_size: int = 16):
        self.bs = block_size
        self.max_seqs = max_seqs
        self.max_blocks = max_blocks_per_seq
        self.free = list(range(num_blocks - 1, -1, -1))   # top of stack = end = block 0
        self.table: dict[int, list[int]] = {}
        self.length: dict[int, int] = {}

    def alloc(self, seq_ids, n_new):
        """Returns the slot mapping (one slot per new token, rows in call order)."""
        if len(seq_ids) != len(n_new) or len(set(seq_ids)) != len(seq_ids):
            raise AllocError("EINVAL")
        need = 0
        for s, n in zip(seq_ids, n_new):
            if not (0 <= s < self.max_seqs) or n < 0:
                raise AllocError("EINVAL")
            L = self.length.get(s, 0)
            if L + n < 1 or L + n > self.max_blocks * self.bs:
                raise AllocError("EINVAL")
            need += -(-(L + n) // self.bs) - -(-L // self.bs)
        if need > len(self.free):
            raise AllocError("ENOBLOCKS")
        slots = []
        for s, n in zip(seq_ids, n_new):
            tab = self.table.setdefault(s, [])
            L = self.length.get(s, 0)
            for pos in range(L, L + n):
                if pos % self.bs == 0:
                    tab.append(self.free.pop())
                slots.append(tab[pos // self.bs] * self.bs + pos % self.bs)
            self.length[s] = L + n
        return slots

    def release(self, seq_id):
        if seq_id not in self.table:
            raise AllocError("ESEQ")
        for blk in reversed(self.table.pop(seq_id)):
            self.free.append(blk)
        del self.length[seq_id]

    def held(self) -> int:
        return sum(len(t) for t in self.table.values())
