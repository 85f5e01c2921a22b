"""Host RadixTrie vs the reference (golden radix_ops from radix.py)."""
from __future__ import annotations

from conftest import load_golden
from paper_2605_26289_b200.kvcache import CapacityExhausted, UnifiedKvCache
from paper_2605_26289_b200.kvcache import PyUnifiedKvCache
from paper_2605_26289_b200.radix import BudgetExceeded, PyRadixTrie, RadixTrie


def test_golden_radix_sequences():
    cases = load_golden("radix_ops.json.gz")
    for case in cases:
        kv = UnifiedKvCache(512)
        trie = RadixTrie(kv, cell_budget=case["budget"])
        for op in case["ops"]:
            err = None
            s = op["seq"]
            try:
                if op["op"] == "save":
                    toks = op["tokens"]
                    held = kv.seq_len(s)
                    if held < len(toks):
                        kv.append_cells(s, len(toks) - held)
                    assert trie.save(toks, s, 0) == op["ret"]
                elif op["op"] == "lookup":
                    m = trie.longest_prefix(op["tokens"])
                    assert {"length": m.length, "runs": [list(r) for r in m.runs],
                            "donor": m.donor} == op["ret"]
                elif op["op"] == "evict":
                    assert trie.evict(op["n"]) == op["ret"]
                else:
                    assert kv.release_sequence(s) == op["ret"]
            except BudgetExceeded:
                err = "BudgetExceeded"
            except CapacityExhausted:
                err = "CapacityExhausted"
            assert err == op["err"]
            assert trie.dump() == op["dump"], op
            assert trie.total_cells == op["cells"]
            assert kv.occupancy == op["occ"]
            assert trie.evicted_cells_total == op["evicted_total"]


def test_eviction_tie_break_lower_first_token():
    # pokes node internals: the Python restatement; the native core is held to
    # it by the differential fuzz (test_host_native.py)
    kv = PyUnifiedKvCache(4096)
    trie = PyRadixTrie(kv, 2048)
    kv.append_cells(1, 4)
    trie.save([5, 5], 1, 0)
    trie.save([3, 3], 1, 2)
    for node in trie.root.children.values():
        node.last_touch = 42
    trie.evict(2)
    assert trie.longest_prefix([3, 3]).length == 0
    assert trie.longest_prefix([5, 5]).length == 2


def test_common_prefix_len_chunked_matches_element_loop():
    """The chunked slice comparison returns the element loop's answer (the
    reference `_common_len`) for every mismatch position, chunk boundaries
    and empty inputs included."""
    import random

    from paper_2605_26289_b200.radix import common_prefix_len

    def loop(a, b):
        n, i = min(len(a), len(b)), 0
        while i < n and a[i] == b[i]:
            i += 1
        return i

    rng = random.Random(3)
    for n in [0, 1, 31, 32, 33, 511, 512, 513, 544, 1100, 4096]:
        a = [rng.randrange(5) for _ in range(n)]
        for k in sorted({0, n // 2, n - 1 if n else 0, n, 32, 512, 543} - {-1}):
            if k > n:
                continue
            b = a[:k] + [9] + a[k:]  # mismatch at k (or b longer by one when k == n)
            assert common_prefix_len(a, b) == loop(a, b) == k
            assert common_prefix_len(b, a) == k
        assert common_prefix_len(a, list(a)) == n
