"""CPU model of K1s (`k_stack_replay`, csrc/cache_sim.cu) against the C
oracle's exact LRU replay (itself pinned to the reference, test_oracle_golden).

K1s replaces the sequential replay by Mattson's stack distance: with no pin
able to bind (capacity C > every row's key count) the reference cache is a
pure LRU over its access sequence, and a touch of x hits iff fewer than C
distinct other keys were accessed since x's previous access. This test runs
the kernel's decision rules row by row in numpy/Python -- same-row prefetch,
the O(1) previous-token formula from prefix sums, the one-token lower bound,
the span unions up to dmax tokens back, the row-level shortcut, the "undecided
-> exact replay" hand-over -- and requires the oracle's cache-hit counters.
It checks the algorithm (the GPU test test_gpu_stack.py checks the kernel)."""
import numpy as np
import pytest


def _lowest(m, n):
    out = 0
    while m and n > 0:
        b = m & -m
        out |= b
        m ^= b
        n -= 1
    return out


def _above(x):
    return ~((2 << x) - 1) & ((1 << 64) - 1)


def _after_last(k, t, x):
    if (t >> x) & 1:
        return t & _above(x)
    return (k & _above(x)) | t


def _stack_prompt(T, P, L, warmup, cap, limit, dmax=4, union_budget=8 * 32):
    """(decided, per-layer hits) of one prompt under K1s's rules."""
    n = len(T)
    K = np.zeros(n, dtype=object)
    S = [0] * n
    for i in range(n):
        k = int(P[i]) if P is not None else 0
        if i // L < warmup:
            k = 0
        if bin(k).count("1") > limit:
            k = _lowest(k, limit)
        K[i] = k
        S[i] = k | int(T[i])
        if bin(S[i]).count("1") >= cap:
            return False, None
    pn = np.cumsum([bin(s).count("1") for s in S])

    def pre(q):
        return 0 if q < 0 else int(pn[q])

    hits = np.zeros(L, dtype=np.int64)
    unions = 0
    for i in range(n):
        t, l = divmod(i, L)
        if t < warmup:
            continue
        Ti, Ki = int(T[i]), int(K[i])
        ch = bin(Ti & Ki).count("1")
        tm = Ti & ~Ki
        if i < L or pre(i - 1) - pre(i - L) >= cap:
            tm = 0  # row-level shortcut: every other touch misses
        while tm:
            x = (tm & -tm).bit_length() - 1
            tm &= tm - 1
            before = Ki | (Ti & ((1 << x) - 1))
            q1 = i - L
            hit = False
            if q1 >= 0 and (S[q1] >> x) & 1:
                D = pre(i - 1) - pre(i - L) + bin(_after_last(int(K[q1]), int(T[q1]), x) | before).count("1")
                hit = D < cap
            elif i - 2 * L >= 0 and pre(i - 1) - pre(i - L - 1) < cap:
                jf, none = 0, False
                for j in range(2, dmax + 1):
                    q = i - j * L
                    if q < 0:
                        none = True
                        break
                    if (S[q] >> x) & 1:
                        jf = j
                        break
                unions += 1
                if not none and unions > union_budget:
                    return False, None
                if not none:
                    j = jf if jf else dmax
                    D = 0
                    for o in range(1, L):
                        u = 0
                        for q in range(i - j * L + o, i, L):
                            u |= S[q]
                        D += bin(u).count("1")
                    u = before
                    for m in range(1, j):
                        u |= S[i - m * L]
                    if jf:
                        u |= _after_last(int(K[i - j * L]), int(T[i - j * L]), x)
                    D += bin(u).count("1")
                    if jf:
                        hit = D < cap
                    elif D < cap and i - (dmax + 1) * L >= 0:
                        return False, None
            ch += int(hit)
        hits[l] += ch
    return True, hits


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("geom", [(6, 16, 3), (4, 64, 6)])
def test_stack_model_matches_oracle(oracle, seed, geom):
    L, E, k = geom
    spec = oracle.GenSpec(12, 40, L, E, k, max(k, E // 4), 0.8, seed)
    truth, _, row_off = oracle.generate_packed(spec, procs=1)
    truth = truth.reshape(-1)
    rng = np.random.default_rng(seed)
    # predictions: the truth of the next token shifted, plus noise, up to 2k experts
    pred = np.zeros_like(truth)
    for r in range(len(truth)):
        bits = rng.choice(E, size=rng.integers(0, 2 * k + 1), replace=False)
        m = 0
        for b in bits:
            m |= 1 << int(b)
        pred[r] = np.uint64(m)
    warmup, budget = 3, k
    n_decided = 0
    for cap in (2 * k + 1, 3 * k, L * k // 2, L * k, 2 * L * k):
        if cap > L * E:
            continue
        want, _, _ = oracle.cache_sim(truth, pred, row_off, L, E, warmup, cap, budget)
        layer_hits = np.zeros(L, dtype=np.int64)
        for p in range(len(row_off) - 1):
            r0, r1 = int(row_off[p]), int(row_off[p + 1])
            ok, h = _stack_prompt(truth[r0:r1], pred[r0:r1], L, warmup, cap, budget)
            if ok:
                n_decided += 1
            else:  # handed to the exact replay: take the oracle's own numbers
                one = np.array([0, r1 - r0], dtype=np.int64)
                c, _, _ = oracle.cache_sim(truth[r0:r1], pred[r0:r1], one, L, E, warmup, cap,
                                           budget)
                h = c[4 + L:4 + 2 * L]
            layer_hits += h
        assert np.array_equal(layer_hits, want[4 + L:4 + 2 * L]), (cap, seed, geom)
        assert int(layer_hits.sum()) == int(want[1])
    assert n_decided > 0
