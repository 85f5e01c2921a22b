/*
 * ORACLE - test infrastructure only.  Nothing in the product path links or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it, and only as the checker.
 *
 * Plain-C restatement of the reference's integer hot kernels
 * (deltaserve._kernels, /root/reference/pkg/src/deltaserve/_kernels/).
 * Pinned against: the reference's own known-answer tests
 * (pkg/tests/test_kernels.py:61-120, test_speculator.py:22-63,
 * test_engine.py:127-141) and against the reference build in oracle/_ref
 * on seeded random inputs (tests/golden/make_golden.py -> kernels.json).
 *
 * Build: gcc -O2 -shared -fPIC -o oracle/libds_oracle.so oracle/ds_oracle.c
 */
#include <stdint.h>
#include <stddef.h>

#define FNV32_OFFSET 0x811C9DC5u
#define FNV32_PRIME 0x01000193u
#define FNV64_OFFSET 0xCBF29CE484222325ull
#define FNV64_PRIME 0x100000001B3ull

/* _native.pyx:18-24 / fallback.py:19-23: FNV-1a 32 over raw bytes. */
uint32_t oracle_fnv1a32_bytes(const uint8_t *p, size_t n) {
    uint32_t h = FNV32_OFFSET;
    for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * FNV32_PRIME;
    return h;
}

/* _native.pyx:27-33 / fallback.py:26-30: FNV-1a 64 over raw bytes. */
uint64_t oracle_fnv1a64_bytes(const uint8_t *p, size_t n) {
    uint64_t h = FNV64_OFFSET;
    for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * FNV64_PRIME;
    return h;
}

/* _native.pyx:36-46 / fallback.py:33-42: tokens hashed as 4 little-endian
 * bytes each (uint32 reinterpretation of int32), seeded by `state`. */
uint32_t oracle_fnv1a32_tokens(const int32_t *tok, size_t n, uint32_t state) {
    uint32_t h = state;
    for (size_t i = 0; i < n; ++i) {
        uint32_t t = (uint32_t)tok[i];
        for (int b = 0; b < 4; ++b) h = (h ^ ((t >> (8 * b)) & 0xFFu)) * FNV32_PRIME;
    }
    return h;
}

/* _native.pyx:49-59 / fallback.py:45-54. */
uint64_t oracle_fnv1a64_tokens(const int32_t *tok, size_t n, uint64_t state) {
    uint64_t h = state;
    for (size_t i = 0; i < n; ++i) {
        uint64_t t = (uint64_t)(uint32_t)tok[i];
        for (int b = 0; b < 4; ++b) h = (h ^ ((t >> (8 * b)) & 0xFFu)) * FNV64_PRIME;
    }
    return h;
}

/* _native.pyx:62-81 / fallback.py:57-80: index e following the most recent
 * earlier occurrence of the trailing min_match-gram (e <= n-1), else -1. */
int64_t oracle_copy_continuation(const int32_t *tok, int64_t n, int64_t mm) {
    if (n <= mm || mm <= 0) return -1;
    const int64_t g = n - mm;
    for (int64_t start = n - mm - 1; start >= 0; --start) {
        int64_t j = 0;
        while (j < mm && tok[start + j] == tok[g + j]) ++j;
        if (j == mm) return start + mm;
    }
    return -1;
}

/* _native.pyx:84-119 / fallback.py:83-120: longest (then most recent)
 * occurrence of a suffix of `tail` (length >= min_len) inside `ring` that
 * leaves at least one following token.  Writes (e, length) or (-1, 0). */
void oracle_longest_suffix_match(const int32_t *ring, int64_t n, const int32_t *tail,
                                 int64_t t, int64_t min_len, int64_t *e_out,
                                 int64_t *len_out) {
    *e_out = -1;
    *len_out = 0;
    if (t < min_len || n <= min_len || min_len <= 0) return;
    const int64_t gs = t - min_len;
    int64_t best_e = -1, best_len = 0;
    for (int64_t start = n - min_len - 1; start >= 0; --start) {
        int64_t j = 0;
        while (j < min_len && ring[start + j] == tail[gs + j]) ++j;
        if (j < min_len) continue;
        const int64_t e = start + min_len;
        const int64_t max_len = t < e ? t : e;
        int64_t len = min_len;
        while (len < max_len && ring[e - len - 1] == tail[t - len - 1]) ++len;
        if (len > best_len) { best_len = len; best_e = e; }
    }
    if (best_e >= 0) { *e_out = best_e; *len_out = best_len; }
}

/* Copy-model greedy token for one query row (engine.py:196-216): copy rule over
 * the full preceding sequence, else FNV-1a64(preceding) mod vocab. */
void oracle_copy_policy(const int32_t *full, int64_t upto, int64_t mm, int64_t vocab,
                        int32_t *token_out, int32_t *source_out) {
    int64_t e = oracle_copy_continuation(full, upto, mm);
    if (e >= 0) {
        *token_out = full[e];
        *source_out = (int32_t)e;
    } else {
        *token_out = (int32_t)(oracle_fnv1a64_tokens(full, (size_t)upto, FNV64_OFFSET) %
                               (uint64_t)vocab);
        *source_out = -1;
    }
}
