"""TEST INFRASTRUCTURE — restatement of the KV page allocator
(paper_2601_11589_b200/csrc/executor.cu: alloc_pages / ensure_capacity /
session_release) used to pin page tables bit-exactly.

Rules: 64-token pages; a session owns ceil(kv_tokens / 64) pages in
allocation order; new pages are taken lowest-free-id first; releasing a
session returns all its pages. A member (session, L, H) needs capacity for
H + L tokens; kv_len becomes max(kv_len, H + L).

Parity: the reference has no KV cache — page tables are
builder-defined; this restatement is the oracle.
"""
from __future__ import annotations

import heapq

PAGE = 64


class PageOracle:
    def __init__(self, n_pages: int):
        self.free = list(range(n_pages))
        heapq.heapify(self.free)
        self.sessions: dict[int, list[int]] = {}
        self.kv_len: dict[int, int] = {}

    def submit(self, members: list[tuple[int, int, int]]) -> None:
        for sid, L, H in members:
            if self.kv_len.get(sid, 0) < H:
                raise ValueError(f"session {sid} history not resident")
            pages = self.sessions.setdefault(sid, [])
            self.kv_len.setdefault(sid, 0)
            need = -(-(H + L) // PAGE)
            while len(pages) < need:
                if not self.free:
                    raise MemoryError("page pool exhausted")
                pages.append(heapq.heappop(self.free))
        for sid, L, H in members:
            self.kv_len[sid] = max(self.kv_len[sid], H + L)

    def release(self, sid: int) -> None:
        for p in self.sessions.pop(sid, []):
            heapq.heappush(self.free, p)
        self.kv_len.pop(sid, None)

    def table(self, sid: int) -> tuple[list[int], int]:
        return list(self.sessions.get(sid, [])), self.kv_len.get(sid, 0)
