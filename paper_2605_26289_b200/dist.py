"""Multi-GPU: sessions shard by id, prefixes migrate between GPUs at admission.

Sessions and agents share nothing but optional radix prefixes, so the unit of
distribution is the session: one process per GPU, each with its own weights
replica, SequencePool, paged KV store, RadixTrie and InferenceCore
(SURVEY.md section 8e).  ``route`` places a session by FNV-1a32 of its id (the
reference's own hash, _native.pyx:18-24).  The reference itself is
single-GPU; nothing here changes a single rank's transcript.

The only data movement between ranks is **prefix migration**, wired into
admission (``InferenceCore._admit``, reference scheduler.py:422-480):

* when a rank commits a prefix to its radix trie (``_finish_slot``) it
  announces the tokens to its peers through the job's key-value store; each
  peer mirrors them in a token-only trie per rank - the prefix directory
  (4 B per token, against 131 KB of K/V per token at the 8B shape);
* when a rank admits a request whose local radix match is shorter than the
  longest common prefix of the prompt with a peer's mirror, it asks that
  peer for the cells past its own match.  The owner
  re-walks its trie (the prefix may have been trimmed or evicted since the
  announcement), replies with the length it actually holds, then sends that
  many cells' K/V rows as ONE [L][2][nkv][n][hd] message on the data group
  (NCCL over NVLink on GPUs; ``ds_kv_pack_cells`` packs them);
* the requester allocates exactly that many cells on a scratch sequence
  (aliasing its own matched prefix in front), receives the message and
  scatters it straight into the new cells with the same kernel
  (``unpack``), commits the prefix to its trie and drops the scratch table.
  The admission then finds the longer radix match and restores it by the
  usual metadata-only alias.

Every rank services its peers' requests between iterations (``poll`` at the
top of each ``step``) and while it waits for a reply of its own, so two ranks
asking each other at once do not deadlock.  ``close`` says goodbye and keeps
serving until every peer has said goodbye too.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch.distributed as dist

FNV32_OFFSET = 0x811C9DC5
FNV32_PRIME = 0x01000193


def _fnv1a32_bytes(data: bytes) -> int:
    """Host routing hash (same function as the reference fnv1a32_bytes)."""
    h = FNV32_OFFSET
    for b in data:
        h = ((h ^ b) * FNV32_PRIME) & 0xFFFFFFFF
    return h


def route(session_id: str, world: int) -> int:
    """Rank that owns a session: fnv1a32(session_id) mod world."""
    return _fnv1a32_bytes(session_id.encode("utf-8")) % max(1, world)


class TokenTrie:
    """Token-only radix trie: a peer's cached prefixes as announced (no cells).
    The requester finds, per peer, the longest common prefix of a prompt with
    anything that peer committed - the same token-granular match the
    reference RadixTrie computes locally (radix.py:81-100), so a partial
    overlap (a shared tool schema under different user turns) is found too."""

    __slots__ = ("seg", "kids")

    def __init__(self, seg=()):
        self.seg = list(seg)
        self.kids: dict[int, TokenTrie] = {}

    def insert(self, tokens) -> None:
        from .radix import common_prefix_len

        node, i, n = self, 0, len(tokens)
        while i < n:
            child = node.kids.get(tokens[i])
            if child is None:
                node.kids[tokens[i]] = TokenTrie(tokens[i:])
                return
            c = common_prefix_len(child.seg, tokens[i:i + len(child.seg)])
            if c < len(child.seg):  # split the child at the divergence
                mid = TokenTrie(child.seg[:c])
                child.seg = child.seg[c:]
                mid.kids[child.seg[0]] = child
                node.kids[tokens[i]] = mid
                child = mid
            node, i = child, i + c

    def longest(self, tokens) -> int:
        from .radix import common_prefix_len

        node, i, n = self, 0, len(tokens)
        while i < n:
            child = node.kids.get(tokens[i])
            if child is None:
                break
            c = common_prefix_len(child.seg, tokens[i:i + len(child.seg)])
            i += c
            if c < len(child.seg):
                break
            node = child
        return i


class PrefixDirectory:
    """What each peer rank has committed to its radix trie (token tries fed by
    announcements).  Entries can be stale - a peer may have evicted since -
    so the owner re-walks its own trie when asked."""

    def __init__(self):
        self.tries: dict[int, TokenTrie] = {}

    def publish(self, rank: int, tokens) -> None:
        self.tries.setdefault(rank, TokenTrie()).insert(list(tokens))

    def best_remote(self, tokens, rank: int, limit: int) -> tuple[int, int]:
        """(peer rank, length) of the longest announced prefix of tokens[:limit]
        held by another rank; (-1, 0) if none."""
        best = (-1, 0)
        head = tokens[:limit]
        for r, trie in self.tries.items():
            if r == rank:
                continue
            ln = trie.longest(head)
            if ln > best[1]:
                best = (r, ln)
        return best


# control messages through the job's key-value store
ANNOUNCE, REQUEST, REPLY, BYE = 1, 2, 3, 4


class PrefixMigrator:
    """Admission-time prefix migration between the ranks of one node.

    Control messages go through the job's TCP key-value store (the
    rendezvous store of ``torch.distributed``): each rank has an inbox - a
    tail counter bumped with ``add`` and one key per message - so ``poll``
    costs one store round trip and never blocks.  (Non-blocking point-to-point
    receives cannot be polled on every backend: a gloo irecv only completes in
    ``wait``.)  The K/V payload goes over ``data_group`` (the default NCCL
    group on GPUs).  One migration runs at a time (a store lock held by the
    requester): the owner answers from inside ``poll`` with a blocking send,
    which can then never meet a send in the opposite direction.  Attach with
    ``PrefixMigrator(core, ...)``; the core then polls, announces and fetches
    by itself.
    """

    def __init__(self, core, data_group=None, store=None, min_gain: int = 32,
                 timeout_s: float = 120.0, namespace: str = "ds_mig"):
        from torch.distributed import distributed_c10d as c10d

        self.core = core
        self.data = data_group
        self.store = store if store is not None else c10d._get_default_store()
        self.ns = namespace
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.peers = [r for r in range(self.world) if r != self.rank]
        self.min_gain = min_gain
        self.timeout_s = timeout_s
        self.directory = PrefixDirectory()
        self._head = 0                       # messages of my inbox consumed
        self._replies: dict[int, int] = {}
        self._bye: set[int] = set()
        self._closed = False
        self.stats = {"fetches": 0, "cells_in": 0, "bytes_in": 0, "seconds_in": 0.0,
                      "served": 0, "cells_out": 0, "bytes_out": 0}
        core.migrator = self

    # -- control plane ---------------------------------------------------------------

    def _send(self, dst: int, kind: int, a: int = 0, tokens=None) -> None:
        """Message = int64 (src, kind, a) header + optional int32 token payload."""
        msg = np.array([self.rank, kind, a], dtype=np.int64).tobytes()
        if tokens is not None:
            msg += np.asarray(tokens, dtype=np.int32).tobytes()
        seq = self.store.add(f"{self.ns}/{dst}/tail", 1)
        self.store.set(f"{self.ns}/{dst}/m{seq}", msg)

    def poll(self) -> None:
        """Drain every control message that has arrived; serve requests."""
        tail = self.store.add(f"{self.ns}/{self.rank}/tail", 0)
        while self._head < tail:
            self._head += 1
            key = f"{self.ns}/{self.rank}/m{self._head}"
            raw = self.store.get(key)
            self.store.delete_key(key)
            src, kind, a = (int(x) for x in np.frombuffer(raw[:24], dtype=np.int64))
            self._handle(src, kind, a, np.frombuffer(raw[24:], dtype=np.int32).tolist())

    def _handle(self, src: int, kind: int, a: int, tokens: list) -> None:
        if kind == ANNOUNCE:
            self.directory.publish(src, tokens)
        elif kind == REQUEST:
            self._serve(src, tokens, a)
        elif kind == REPLY:
            self._replies[src] = a
        elif kind == BYE:
            self._bye.add(src)
        else:
            raise RuntimeError(f"unknown migration message {kind} from rank {src}")

    def _lock(self, deadline: float) -> None:
        me = str(self.rank + 1).encode()
        while True:
            cur = self.store.compare_set(f"{self.ns}/lock", "", me)
            if cur == me:
                return
            self.poll()  # the holder may be waiting on us
            if time.monotonic() > deadline:
                raise TimeoutError("prefix migration lock not acquired")
            time.sleep(0.0005)

    def _unlock(self) -> None:
        self.store.set(f"{self.ns}/lock", "")

    # -- announcements (radix save) -----------------------------------------------

    def publish(self, tokens) -> None:
        """A prefix was committed to the local trie: announce it to the peers."""
        if not tokens or self._closed:
            return
        for dst in self.peers:
            self._send(dst, ANNOUNCE, len(tokens), tokens)

    # -- owner side ------------------------------------------------------------------

    def _serve(self, dst: int, tokens: list, start: int) -> None:
        """Send the cells of tokens[start:n], n = what the local trie still
        holds of `tokens` (it may have evicted since announcing)."""
        core = self.core
        m = core.radix.longest_prefix(tokens)
        n = m.length
        n_send = max(0, n - start)
        self._send(dst, REPLY, n if n_send else 0)
        if n_send:
            cells: list[int] = []
            for s_, ln in m.runs:
                cells.extend(range(s_, s_ + ln))
            buf = core.engine.pack_cells(cells[start:n])
            dist.send(buf, dst, group=self.data)
            self.stats["served"] += 1
            self.stats["cells_out"] += n_send
            self.stats["bytes_out"] += buf.numel() * buf.element_size()

    # -- requester side (called from _admit, under the core lock) --------------------

    def fetch(self, prompt, local_match) -> int:
        """If a peer holds a longer prefix of `prompt` than the local radix
        match, migrate the missing cells into the local trie.  Returns the
        number of cells received (0: nothing to gain / nothing held)."""
        from .kvcache import slice_runs
        from .radix import BudgetExceeded

        core = self.core
        n_p = len(prompt)
        limit = n_p - 1  # admission recomputes the last prompt token (scheduler.py:436)
        owner, length = self.directory.best_remote(prompt, self.rank, limit)
        start = local_match.length
        if owner < 0 or length - start < self.min_gain:
            return 0
        kv, seq = core.kv, core.scratch_seq
        kv.release_sequence(seq)
        buf = None
        try:
            if start:  # hold the local match: an eviction below must not free it
                kv.alias_runs(seq, slice_runs(local_match.runs, 0, start))
            if not core._ensure_capacity(length - start):
                return 0
            t0 = time.perf_counter()
            deadline = time.monotonic() + self.timeout_s
            self._lock(deadline)
            try:
                self._replies.pop(owner, None)
                self._send(owner, REQUEST, start, prompt[:length])
                while owner not in self._replies:
                    self.poll()
                    if time.monotonic() > deadline:
                        raise TimeoutError(f"rank {owner} did not answer a prefix request")
                    time.sleep(0.0002)
                n = self._replies.pop(owner)  # what the owner still holds (<= length)
                if n <= start:
                    return 0
                kv.append_cells(seq, n - start)
                cells = kv.cell_ids(seq, start, n)
                buf = core.engine.payload_buffer(n - start)
                dist.recv(buf, owner, group=self.data)
            finally:
                self._unlock()
            core.engine.unpack_cells(cells, buf)
            try:
                core.radix.save(list(prompt[:n]), seq, 0)
            except BudgetExceeded:
                return 0
        finally:
            kv.release_sequence(seq)
        self.stats["fetches"] += 1
        self.stats["cells_in"] += n - start
        self.stats["bytes_in"] += buf.numel() * buf.element_size()
        self.stats["seconds_in"] += time.perf_counter() - t0
        return n - start

    # -- shutdown --------------------------------------------------------------------

    def close(self, timeout_s: float = 300.0) -> None:
        """Say goodbye; keep serving until every peer has said goodbye."""
        if self._closed:
            return
        self._closed = True
        for dst in self.peers:
            self._send(dst, BYE)
        deadline = time.monotonic() + timeout_s
        while len(self._bye) < len(self.peers):
            self.poll()
            if time.monotonic() > deadline:
                raise TimeoutError("peers did not close the migration channel")
            time.sleep(0.001)
        self.core.migrator = None
