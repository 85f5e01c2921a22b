"""Multi-GPU: sessions shard by id, prefixes migrate between GPUs over NCCL.

Sessions and agents share nothing but optional radix prefixes, so the unit of
distribution is the session: one process per GPU, each with its own weights
replica, SequencePool, paged KV store, RadixTrie and InferenceCore
(SURVEY.md section 8e).  ``route`` places a session by FNV-1a32 of its id (the
reference's own hash, _native.pyx:18-24).  The only device collective on the
path is prefix migration: when a peer holds a longer cached prefix (e.g. a
shared tool-schema preamble), the owner packs the prefix's K/V cell rows
(all layers, K and V, head-major) into one buffer and sends it; the receiver
allocates fresh cells, receives straight into that buffer, scatters it into
its pool and commits the prefix to its radix trie - after which restoring it
is the usual metadata-only alias.  A host-side directory of (rank, digest,
length) rides on the torch.distributed object collectives.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
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


@dataclass(frozen=True)
class PrefixEntry:
    rank: int
    digest: int
    length: int


class PrefixDirectory:
    """Which rank caches which prefix (digest = host FNV-1a64 of the tokens)."""

    def __init__(self):
        self.entries: dict[int, PrefixEntry] = {}

    def publish_local(self, rank: int, prefixes: list[tuple[int, int]]) -> None:
        for digest, length in prefixes:
            cur = self.entries.get(digest)
            if cur is None or length > cur.length:
                self.entries[digest] = PrefixEntry(rank, digest, length)

    def sync(self, group=None) -> None:
        """All-gather every rank's entries (CPU object collective)."""
        if not dist.is_initialized() or dist.get_world_size(group) == 1:
            return
        gathered = [None] * dist.get_world_size(group)
        dist.all_gather_object(gathered, list(self.entries.values()), group=group)
        for lst in gathered:
            for e in lst:
                self.publish_local(e.rank, [(e.digest, e.length)])

    def owner(self, digest: int) -> PrefixEntry | None:
        return self.entries.get(digest)


# ---------------------------------------------------------------------------
# cell row packing (head-major pool [L][nkv][cells][hd])
# ---------------------------------------------------------------------------

def pack_cells(k_pool: torch.Tensor, v_pool: torch.Tensor, cells) -> torch.Tensor:
    """[L][2][nkv][n][hd] contiguous buffer of the given cells' K and V rows."""
    idx = torch.as_tensor(list(cells), dtype=torch.long, device=k_pool.device)
    return torch.stack([k_pool.index_select(2, idx), v_pool.index_select(2, idx)], dim=1)


def unpack_cells(k_pool: torch.Tensor, v_pool: torch.Tensor, cells, buf: torch.Tensor) -> None:
    idx = torch.as_tensor(list(cells), dtype=torch.long, device=k_pool.device)
    k_pool.index_copy_(2, idx, buf[:, 0])
    v_pool.index_copy_(2, idx, buf[:, 1])


def send_prefix(k_pool, v_pool, cells, dst: int, group=None) -> int:
    """Send the rows of `cells` to rank dst; returns bytes sent."""
    buf = pack_cells(k_pool, v_pool, cells)
    dist.send(buf, dst, group=group)
    return buf.numel() * buf.element_size()


def recv_prefix(k_pool, v_pool, cells, src: int, group=None) -> int:
    """Receive rows from rank src straight into a buffer and scatter them into
    the freshly allocated `cells`; returns bytes received."""
    L, nkv, _, hd = k_pool.shape
    buf = torch.empty((L, 2, nkv, len(cells), hd), dtype=k_pool.dtype, device=k_pool.device)
    dist.recv(buf, src, group=group)
    unpack_cells(k_pool, v_pool, cells, buf)
    return buf.numel() * buf.element_size()


# ---------------------------------------------------------------------------
# core-level export / import
# ---------------------------------------------------------------------------

def export_prefix(core, tokens) -> list[int]:
    """Physical cells backing the longest cached prefix of tokens (radix walk)."""
    m = core.radix.longest_prefix(tokens)
    cells: list[int] = []
    for s, ln in m.runs:
        cells.extend(range(s, s + ln))
    return cells


def import_prefix(core, tokens, receive) -> int:
    """Allocate cells for `tokens` on a scratch sequence, fill them with
    ``receive(cells)`` (device copy / NCCL recv), commit them to the radix and
    drop the scratch table - the trie's references keep the cells alive, and a
    later request restores them by metadata-only aliasing.  Returns cells."""
    seq = core.scratch_seq
    n = len(tokens)
    core.kv.release_sequence(seq)
    core.kv.append_cells(seq, n)
    cells = core.kv.cell_ids(seq, 0, n)
    receive(cells)
    core.radix.save(list(tokens), seq, 0)
    core.kv.release_sequence(seq)
    return n


def migrate_prefix(src_core, dst_core, tokens, src_rank: int, dst_rank: int, group=None) -> int:
    """Collective prefix migration between two ranks (both call it)."""
    rank = dist.get_rank(group)
    if rank == src_rank:
        cells = export_prefix(src_core, tokens)[: len(tokens)]
        eng = src_core.engine
        return send_prefix(eng.k_pool, eng.v_pool, cells, dst_rank, group)
    if rank == dst_rank:
        eng = dst_core.engine
        nbytes = [0]

        def receive(cells):
            nbytes[0] = recv_prefix(eng.k_pool, eng.v_pool, cells, src_rank, group)

        import_prefix(dst_core, tokens, receive)
        return nbytes[0]
    return 0
