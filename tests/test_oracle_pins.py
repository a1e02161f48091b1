"""Pins for the CPU oracle (oracle/): each test fixes the oracle against something
other than itself -- values the paper/SPEC print, hand-derived fixtures, closed
forms, invariants, brute force on tiny inputs.  CPU only."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from conftest import golden


def hx(vals):
    return np.array([int(v, 16) for v in vals], dtype=np.uint8)


def rand_images(m, Lstar, seed):
    # data from the shared seeded generator, NOT from the oracle
    return [synth.fill(seed, j, 0, Lstar) for j in range(m)]


# ---------------------------------------------------------------- generator ----
def test_splitmix64_published_sequence():
    # SplitMix64 seeded with 0 emits mix(k*gamma): published first outputs
    g = 0x9E3779B97F4A7C15
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    for k, w in enumerate(want):
        assert oracle.splitmix64((k * g) % 2**64) == w
        assert synth.splitmix64((k * g) % 2**64) == w


@pytest.mark.parametrize("nbytes,begin", [(1, 0), (7, 0), (1003, 0), (64, 13)])
def test_generator_copies_agree(nbytes, begin):
    full = synth.fill(12670, 5, 9, nbytes + begin)
    assert np.array_equal(oracle.fill(12670, 5, 9, nbytes, begin), full[begin:])


# ---------------------------------------------------------------- layout (O1/O2) --
def test_layout_golden():
    g = golden("layout_a256.txt")
    sizes = [int(x) for x in g["sizes"][0]]
    off, L = oracle.layout(sizes, 256)
    assert off == [int(x) for x in g["offsets"][0]]
    assert L == int(g["L"][0][0])
    for m, u, Ls, ue in g["common"]:
        assert oracle.common_length([1280, 768, 1024][: int(m)], int(u)) == (int(Ls), int(ue))
    assert oracle.common_length([1280], 64) == (1280, 64)


def test_layout_brute_force_properties():
    rng = np.random.default_rng(0)
    for _ in range(50):
        sizes = rng.integers(1, 2000, size=int(rng.integers(1, 12))).tolist()
        off, L = oracle.layout(sizes, 256)
        # aligned, ordered, non-overlapping, minimal gaps (< 256), L covers all
        for t in range(len(sizes)):
            assert off[t] % 256 == 0
            if t:
                prev_end = off[t - 1] + sizes[t - 1]
                assert prev_end <= off[t] < prev_end + 256
        assert L % 256 == 0 and off[-1] + sizes[-1] <= L < off[-1] + sizes[-1] + 256


# ---------------------------------------------------------------- pack / unpack --
def test_pack_unpack_roundtrip_and_zero_pad():
    sizes = [3, 300, 1, 256, 4097]
    ts = [synth.fill(1, 0, t, n) for t, n in enumerate(sizes)]
    off, L = oracle.layout(sizes, 256)
    Lstar = L + 512
    D = oracle.pack(ts, off, Lstar)
    # every byte not covered by a tensor is zero (I3)
    covered = np.zeros(Lstar, dtype=bool)
    for o, n in zip(off, sizes):
        covered[o:o + n] = True
    assert not D[~covered].any()
    # independent check of placement with numpy slicing
    for t, (o, n) in enumerate(zip(off, sizes)):
        assert np.array_equal(D[o:o + n], ts[t])
    back = oracle.unpack(D, sizes, off)
    for a, b in zip(back, ts):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- encode (O4) ----
@pytest.mark.parametrize("name", ["aec_m3_u1.txt", "aec_m4_eq1.txt"])
def test_encode_hand_derived_golden(name):
    g = golden(name)
    m, u = int(g["m"][0][0]), int(g["u"][0][0])
    Ds = [hx(g[f"D{j}"][0]) for j in range(m)]
    for r in range(m):
        assert np.array_equal(oracle.encode(Ds, u, r), hx(g[f"P{r}"][0])), f"row {r}"


def test_eq1_row0_is_b0_c0_d0():
    # PAPER.md Eq 1 (P.476): p_bcd0 = b0 ^ c0 ^ d0, at every u and every stripe
    rng = np.random.default_rng(3)
    for u in (1, 4, 16):
        Ds = [rng.integers(0, 256, 3 * u * 5, dtype=np.uint8) for _ in range(4)]
        P0 = oracle.encode(Ds, u, 0)
        for s in range(5):
            unit = lambda j: Ds[j][s * 3 * u: s * 3 * u + u]
            assert np.array_equal(P0[s * u:(s + 1) * u], unit(1) ^ unit(2) ^ unit(3))


def test_spec_codec_vectors():
    g = golden("spec_codec_vectors.txt")
    b0, c0, d0 = hx(g["encode_in"][0])
    Ds = [np.array([0x5C], np.uint8), np.array([b0]), np.array([c0]), np.array([d0])]
    Ds = [np.concatenate([d, np.zeros(2, np.uint8)]) for d in Ds]  # m=4, u=1, L*=3
    assert oracle.encode(Ds, 1, 0)[0] == hx(g["encode_out"][0])[0]
    # decode: lose rank 1 (b): b0 = p ^ c0 ^ d0 (S.336)
    Ps = oracle.encode_all(Ds, 1)
    Dk = oracle.rebuild([Ds[0], None, Ds[2], Ds[3]], [Ps[0], None, Ps[2], Ps[3]], 1, 1)
    assert Dk[0] == hx(g["decode_out"][0])[0]
    # m=3: parity of row 0 is b0 ^ c0; survivor b0 -> c0 (S.337)
    D3 = [np.array([1, 2, 3, 4], np.uint8), np.array([7, 8, 9, 10], np.uint8), np.array([200, 100, 50, 25], np.uint8)]
    P3 = oracle.encode_all(D3, 1)
    assert P3[0][0] == D3[1][0] ^ D3[2][0]
    assert np.array_equal(oracle.rebuild([D3[0], D3[1], None], [P3[0], P3[1], None], 1, 2), D3[2])


def test_m2_is_arc_mirror():
    # I5: m=2 -> each rank's parity is the other's data (ARC volume 2W_n/m, P.459, S.317)
    Ds = rand_images(2, 4096, 7)
    for u in (1, 64, 0):
        Lstar, ue = oracle.common_length([4096, 4096], u)
        P0, P1 = oracle.encode(Ds, ue, 0), oracle.encode(Ds, ue, 1)
        assert np.array_equal(P0, Ds[1]) and np.array_equal(P1, Ds[0])


def test_parity_volume_closed_form():
    # I4: |P_r| = W_n/(m(m-1)) for divisible sizes (P.486; S.328: W_n=1200, m=4 -> 100)
    W_n, m = 1200, 4
    Ls = [W_n // m] * m
    off, L = oracle.layout([W_n // m], 4)
    assert L == 300
    Lstar, u = oracle.common_length(Ls, 100)
    Ds = rand_images(m, Lstar, 11)
    for r in range(m):
        assert oracle.encode(Ds, u, r).size == W_n // (m * (m - 1)) == 100


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6])
def test_single_bit_flip_hits_exactly_one_parity_bit(m):
    # I11: every data bit is covered by exactly one parity bit, held by a rank other
    # than its owner (so any single loss is recoverable).  A transposed sigma, a
    # dropped term or a wrong unit index all fail this.
    for u in (1, 3):
        Lstar = (m - 1) * u * 2
        Ds = rand_images(m, Lstar, 100 + m)
        base = oracle.encode_all(Ds, u)
        for j in range(m):
            for b in range(Lstar):
                bit = 1 << ((b * 7 + j) % 8)
                D2 = [d.copy() for d in Ds]
                D2[j][b] ^= bit
                diffs = [(r, i, int(x ^ y)) for r, P in enumerate(oracle.encode_all(D2, u))
                         for i, (x, y) in enumerate(zip(P, base[r])) if x != y]
                assert len(diffs) == 1 and diffs[0][2] == bit and diffs[0][0] != j


def test_linearity():
    # I7: enc(D ^ D') = enc(D) ^ enc(D'); enc(0) = 0  (S.371)
    m, u, L = 5, 4, 4 * 4 * 3
    A, B = rand_images(m, L, 1), rand_images(m, L, 2)
    for r in range(m):
        assert np.array_equal(oracle.encode([a ^ b for a, b in zip(A, B)], u, r),
                              oracle.encode(A, u, r) ^ oracle.encode(B, u, r))
        assert not oracle.encode([np.zeros(L, np.uint8)] * m, u, r).any()


def test_stripe_locality_bucket_invariance():
    # I8: parity of a prefix of whole stripes = prefix of the whole-stream parity
    m, u = 4, 8
    L = (m - 1) * u * 10
    Ds = rand_images(m, L, 5)
    for r in range(m):
        full = oracle.encode(Ds, u, r)
        for ns in (1, 3, 7):
            part = oracle.encode([d[: ns * (m - 1) * u] for d in Ds], u, r)
            assert np.array_equal(part, full[: ns * u])


# ---------------------------------------------------------------- rebuild (O6) --
@pytest.mark.parametrize("m", [2, 3, 4, 5, 6, 8])
def test_rebuild_every_lost_rank_exact(m):
    # I2: any single lost rank rebuilds exactly (P.460 "no more than one node failure",
    # P.486 "reliability of AEC is the same as ARC"); expected = generator output
    for u in (1, 2, 4, 16):
        Lstar = (m - 1) * u * 3
        Ds = rand_images(m, Lstar, 40 + m * u)
        Ps = oracle.encode_all(Ds, u)
        for k in range(m):
            surv_D = [None if j == k else Ds[j] for j in range(m)]
            surv_P = [None if j == k else Ps[j] for j in range(m)]
            lost = [j == k for j in range(m)]
            assert np.array_equal(oracle.rebuild(surv_D, surv_P, u, k, lost), Ds[k])


def test_rebuild_row_xor_zero():
    # I1: XOR of a row's data units and its parity is zero; checked by brute force
    # over all (rank, unit) pairs assigned to a row via the coverage test above.
    m, u = 5, 2
    Lstar = (m - 1) * u * 2
    Ds = rand_images(m, Lstar, 9)
    Ps = oracle.encode_all(Ds, u)
    total = np.zeros(u, np.uint8)
    for s in range(2):
        acc = np.zeros(u, np.uint8)
        for r in range(m):
            acc ^= Ps[r][s * u:(s + 1) * u]
        for j in range(m):
            for i in range(m - 1):  # every data unit of the stripe appears in exactly one row
                acc ^= Ds[j][s * (m - 1) * u + i * u: s * (m - 1) * u + (i + 1) * u]
        total |= acc
    assert not total.any()


def test_two_losses_unrecoverable():
    # I10 (P.460, S.334, S.559); m = 1 has no redundancy (S.314)
    Ds = rand_images(4, 12, 1)
    Ps = oracle.encode_all(Ds, 1)
    with pytest.raises(oracle.OracleError, match="unrecoverable"):
        oracle.rebuild([None, None, Ds[2], Ds[3]], [None, None, Ps[2], Ps[3]], 1, 0,
                       [True, True, False, False])
    with pytest.raises(oracle.OracleError, match="unrecoverable"):
        oracle.rebuild([Ds[0]], [Ps[0]], 1, 0)


# ---------------------------------------------------------------- ARC / collaborative (f2)
def test_arc_ring_placement_and_volume():
    # S.313-318: node i also snapshots node (i+1) mod m; the copies cover every shard
    # exactly once; per-node volume 2 W_n/m (W_n=1000, m=4 -> 500); m=2 -> each holds W_n
    for m in range(2, 9):
        held = sorted((i + 1) % m for i in range(m))
        assert held == list(range(m))
        assert all(oracle.arc_holder(m, (i + 1) % m) == i for i in range(m))
    W_n, m = 1000, 4
    Ds = rand_images(m, W_n // m, 3)
    for i in range(m):
        copy = oracle.arc_copy(Ds, i)
        assert np.array_equal(copy, Ds[(i + 1) % m])
        assert Ds[i].size + copy.size == 2 * W_n // m == 500
    D2 = rand_images(2, 500, 4)
    assert D2[0].size + oracle.arc_copy(D2, 0).size == 1000


def _group(m, u, seed):
    Lstar = (m - 1) * u * 3
    Ds = rand_images(m, Lstar, seed)
    Ps = oracle.encode_all(Ds, u)
    MDs = [oracle.arc_copy(Ds, i) for i in range(m)]
    MPs = [Ps[(i + 1) % m] for i in range(m)]  # ARC+AEC: the neighbour's parity row too (Q20)
    return Ds, Ps, MDs, MPs


def _lose(arrs, lost):
    return [[None if lost[j] else a for j, a in enumerate(arr)] for arr in arrs]


@pytest.mark.parametrize("m", [3, 4, 5, 6])
def test_collaborative_tolerates_every_pair(m):
    # P.507-508 / S.364-366: ARC + AEC together restore any N = 2 failures (m >= 3),
    # bit-exactly (data and parity rows) -- brute force over every pair
    u = 2
    Ds, Ps, MDs, MPs = _group(m, u, 50 + m)
    for a, b in itertools.combinations(range(m), 2):
        lost = [j in (a, b) for j in range(m)]
        out = oracle.recover(oracle.SCHEME_ARC_AEC, lost, *_lose((Ds, Ps, MDs, MPs), lost), u)
        for x in (a, b):
            assert np.array_equal(out[x][0], Ds[x]) and np.array_equal(out[x][1], Ps[x]), (a, b, x)


@pytest.mark.parametrize("m", [2, 3, 4, 6])
def test_single_strategy_tolerates_one(m):
    # S.364-365: ARC alone and AEC alone restore any single failure; each fails on some
    # pair (AEC on every pair, ARC on an adjacent pair); three losses are never restored
    u = 4
    Ds, Ps, MDs, MPs = _group(m, u, 90 + m)
    for x in range(m):
        lost = [j == x for j in range(m)]
        for scheme in (oracle.SCHEME_ARC, oracle.SCHEME_AEC, oracle.SCHEME_ARC_AEC):
            out = oracle.recover(scheme, lost, *_lose((Ds, Ps, MDs, MPs), lost), u)
            assert np.array_equal(out[x][0], Ds[x])
    lost = [j in (0, 1) for j in range(m)]
    for scheme in (oracle.SCHEME_ARC, oracle.SCHEME_AEC):
        with pytest.raises(oracle.OracleError, match="unrecoverable"):
            oracle.recover(scheme, lost, *_lose((Ds, Ps, MDs, MPs), lost), u)
    if m >= 4:  # ARC alone does restore a non-adjacent pair
        lost = [j in (0, 2) for j in range(m)]
        out = oracle.recover(oracle.SCHEME_ARC, lost, *_lose((Ds, Ps, MDs, MPs), lost), u)
        assert np.array_equal(out[0][0], Ds[0]) and np.array_equal(out[2][0], Ds[2])
    if m >= 3:
        lost = [j in (0, 1, 2) for j in range(m)]
        with pytest.raises(oracle.OracleError, match="unrecoverable"):
            oracle.recover(oracle.SCHEME_ARC_AEC, lost, *_lose((Ds, Ps, MDs, MPs), lost), u)


def test_collaborative_needs_mirrored_parity():
    # why reading Q20 mirrors the parity row: without it an adjacent pair (a, a+1) leaves
    # unit sigma(a, a+1) of every stripe of a+1 uncovered -- show that unit is exactly
    # the one the other rows cannot provide
    m, u = 4, 1
    Ds, Ps, MDs, MPs = _group(m, u, 7)
    lost = [True, True, False, False]
    out = oracle.recover(oracle.SCHEME_ARC_AEC, lost, *_lose((Ds, Ps, MDs, MPs), lost), u)
    assert np.array_equal(out[1][0], Ds[1])
    bad_MPs = [None, None, MPs[2], np.zeros_like(MPs[3])]  # member 3 holds member 0's parity: zeroed
    out = oracle.recover(oracle.SCHEME_ARC_AEC, lost, Ds[:0] + [None, None, Ds[2], Ds[3]],
                         [None, None, Ps[2], Ps[3]], [None, None, MDs[2], MDs[3]], bad_MPs, u)
    diff = np.nonzero(out[1][0] != Ds[1])[0]
    stripe = (m - 1) * u
    # only bytes of unit sigma(0, 1) = 0 of each stripe of member 1 are wrong
    assert diff.size and all(d % stripe < u for d in diff)


# ---------------------------------------------------------------- AOR (f4) ----
# Eq 4 (PAPER.md P.502-504): W^(t+1) = W^t - eta * grad^t; reading Q22: fp32, the product
# rounded before the subtraction; bf16 gradients widened exactly.
def test_aor_closed_form_exact_steps():
    # every intermediate is a dyadic rational with few bits: exact in fp32
    w = np.array([1.0, -3.5, 0.0, 1024.0], np.float32)
    g = np.array([0.5, -0.25, 2.0, 8.0], np.float32)
    for t in range(1, 9):
        w = oracle.aor_update(w, g, 0.25)
        assert w.tolist() == [1.0 - 0.125 * t, -3.5 + 0.0625 * t, -0.5 * t, 1024.0 - 2.0 * t]


def test_aor_product_rounded_before_subtraction():
    # eta = g = 1 + 2^-12: eta*g = 1 + 2^-11 + 2^-24 rounds (tie to even) to 1 + 2^-11,
    # so w = 1 + 2^-11 gives exactly 0; a fused multiply-add would give -2^-24.
    x = np.float32(1.0 + 2.0**-12)
    w = np.array([1.0 + 2.0**-11], np.float32)
    out = oracle.aor_update(w, np.array([x], np.float32), float(x))
    assert out[0] == 0.0 and not np.signbit(out[0])


def test_aor_matches_numpy_float32_per_op():
    rng = np.random.default_rng(7)
    w = rng.standard_normal(4099).astype(np.float32)
    g = (rng.standard_normal(4099) * 1e-3).astype(np.float32)
    for eta in (1e-3, 0.1, 3.0e-4, 1.0):
        e32 = np.float32(eta)
        want = w - (e32 * g)          # numpy float32 ops: each rounded to fp32
        assert np.array_equal(oracle.aor_update(w, g, eta).view(np.uint32), want.view(np.uint32))


def test_aor_bf16_gradient_widening():
    import torch
    bits = np.array([0x3F80, 0xC000, 0x4049, 0x0000, 0x8000, 0x0001, 0x7F7F, 0x3C23, 0xBE4D], np.uint16)
    # bf16 -> fp32 through torch's own conversion (an independent library routine)
    gf = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).float().numpy()
    assert gf[:3].tolist() == [1.0, -2.0, 3.140625]
    w = np.linspace(-2, 2, bits.size).astype(np.float32)
    for eta in (0.5, 1e-3):
        assert np.array_equal(oracle.aor_update(w, bits, eta).view(np.uint32),
                              oracle.aor_update(w, gf.astype(np.float32), eta).view(np.uint32))


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5])
def test_aor_recover_brute_force_masks(m):
    rng = np.random.default_rng(m)
    sizes = [int(rng.integers(0, 9)) for _ in range(m)]
    masters0 = [rng.standard_normal(n).astype(np.float32) for n in sizes]
    replicas0 = [masters0[(j + 1) % m].copy() for j in range(m)]   # ring: j holds j+1 (SPEC S.313)
    for mask in range(1, 1 << m):
        lost = [(mask >> j) & 1 for j in range(m)]
        ms = [np.full(sizes[j], np.nan, np.float32) if lost[j] else masters0[j] for j in range(m)]
        rs = [np.full(sizes[(j + 1) % m], np.nan, np.float32) if lost[j] else replicas0[j] for j in range(m)]
        adjacent = any(lost[j] and lost[(j - 1) % m] for j in range(m))
        if m == 1 or adjacent:
            with pytest.raises(oracle.OracleError, match="unrecoverable"):
                oracle.aor_recover(lost, ms, rs)
            continue
        got_m, got_r = oracle.aor_recover(lost, ms, rs)
        for j in range(m):
            assert np.array_equal(got_m[j], masters0[j]) and np.array_equal(got_r[j], replicas0[j])
