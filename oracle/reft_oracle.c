/*
 * oracle/reft_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain, slow, obviously-correct CPU oracle for REFT's snapshot-and-protect hot
 * path (arXiv 2310.12670, "REFT"): pack (snapshot image), AEC XOR parity encode,
 * single-loss rebuild (decode) and unpack (load); ARC copies and two-loss recovery;
 * AOR's Eq 4 replica update and recovery.  Scalar loops only, no
 * blocking, no vectorisation, no threads.  It shares no code, header, table or
 * constant with the CUDA path in paper_2310_12670_b200/ and neither side
 * includes the other.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.
 *
 * Citations: "P.n" = /root/reference/PAPER.md line n, "S.n" = SPEC.md line n,
 * "Q#" = a reading listed in DESIGN.md section 3.
 *
 * Every function returns 0 on success and a negative value on bad arguments.
 * Pins (tests/test_oracle_pins.py): Eq 1 row-0 pattern, SPEC byte vectors,
 * the hand-derived golden fixtures in tests/golden/, m=2 mirror (ARC),
 * exact rebuild of every lost rank from independently generated data,
 * single-bit-flip coverage, linearity, volumes.  No function is "parity unpinned".
 */
#include <stdint.h>
#include <stddef.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL (-1)
#define ORACLE_EUNRECOVERABLE (-2)

static uint64_t align_up(uint64_t x, uint64_t a) { return a ? ((x + a - 1) / a) * a : x; }

/* O1 layout (Q6: registration order, each tensor at an A-aligned offset,
 * zero gaps).  off[t+1] = align_up(off[t] + nbytes[t], A); L = align_up(end, A).
 * The paper is silent on packing order (it copies per tensor, P.662). */
int oracle_layout(uint64_t n, const uint64_t *nbytes, uint64_t align,
                  uint64_t *off, uint64_t *L)
{
    uint64_t end = 0, t;
    if (align == 0 || !L || (n && (!nbytes || !off))) return ORACLE_EINVAL;
    for (t = 0; t < n; t++) {
        off[t] = align_up(end, align);
        end = off[t] + nbytes[t];
    }
    *L = align_up(end, align);
    return ORACLE_OK;
}

/* O2 common packed length L* (Q4, Q5).  Every member of the group is zero-padded
 * to one length that is a whole number of stripes of (m-1) units of u bytes.
 * u = 0 is SPEC's whole-shard split into m-1 sub-slices (S.378): one stripe,
 * u = L* /(m-1) with L* a multiple of (m-1)*256.  m = 1: no protection, L* = L_0. */
int oracle_common_length(uint64_t m, const uint64_t *Lj, uint64_t u,
                         uint64_t *Lstar, uint64_t *u_eff)
{
    uint64_t mx = 0, j;
    if (m < 1 || !Lj || !Lstar || !u_eff) return ORACLE_EINVAL;
    for (j = 0; j < m; j++) if (Lj[j] > mx) mx = Lj[j];
    if (m == 1) { *Lstar = Lj[0]; *u_eff = u; return ORACLE_OK; }
    if (u == 0) {
        *Lstar = align_up(mx, (m - 1) * 256);
        *u_eff = *Lstar / (m - 1);
    } else {
        *Lstar = align_up(mx, (m - 1) * u);
        *u_eff = u;
    }
    return ORACLE_OK;
}

/* O3 pack: D = zeros(L*); D[off[t] : off[t]+nbytes[t]] = tensor t's bytes.
 * This is the "snapshot" image of one rank's shard (P.553 "ongoing snapshot
 * accepts flushed parameters from device memory"). */
int oracle_pack(uint64_t n, const uint8_t *const *src, const uint64_t *nbytes,
                const uint64_t *off, uint64_t Lstar, uint8_t *D)
{
    uint64_t i, t;
    if (!D && Lstar) return ORACLE_EINVAL;
    for (i = 0; i < Lstar; i++) D[i] = 0;
    for (t = 0; t < n; t++) {
        if (off[t] + nbytes[t] > Lstar) return ORACLE_EINVAL;
        for (i = 0; i < nbytes[t]; i++) D[off[t] + i] = src[t][i];
    }
    return ORACLE_OK;
}

/* O7 unpack (load): tensor t's bytes = D[off[t] : off[t]+nbytes[t]] (P.545 step 1,
 * "load its checkpoint shard from local Host memory"). */
int oracle_unpack(uint64_t n, uint8_t *const *dst, const uint64_t *nbytes,
                  const uint64_t *off, uint64_t Lstar, const uint8_t *D)
{
    uint64_t i, t;
    for (t = 0; t < n; t++) {
        if (off[t] + nbytes[t] > Lstar) return ORACLE_EINVAL;
        for (i = 0; i < nbytes[t]; i++) dst[t][i] = D[off[t] + i];
    }
    return ORACLE_OK;
}

/* sigma(r, j) = r - [r > j]: the index of the unit of rank j's stripe that row r
 * protects (Q3).  Row 0 at m = 4 gives units (b0, c0, d0) = Eq 1, P.476. */
static uint64_t sigma(uint64_t r, uint64_t j) { return r - (r > j ? 1 : 0); }

/* O4 AEC encode (Eq 1, P.474-477; sub-slicing P.486, S.378; rotation Q3, Q4).
 * For every stripe s in [0, L* /((m-1)u)) and byte i in [0, u):
 *   P_r[s*u + i] = XOR_{j != r} D_j[s*(m-1)*u + sigma(r, j)*u + i]
 * D[j] is rank j's packed image of L* bytes; P receives L* /(m-1) bytes. */
int oracle_encode(uint64_t m, const uint8_t *const *D, uint64_t Lstar, uint64_t u,
                  uint64_t r, uint8_t *P)
{
    uint64_t s, i, j, nstripes;
    if (m < 2 || u == 0 || r >= m || !D || !P) return ORACLE_EINVAL;
    if (Lstar % ((m - 1) * u)) return ORACLE_EINVAL;
    nstripes = Lstar / ((m - 1) * u);
    for (s = 0; s < nstripes; s++) {
        for (i = 0; i < u; i++) {
            uint8_t acc = 0;
            for (j = 0; j < m; j++) {
                if (j == r) continue;
                acc ^= D[j][s * (m - 1) * u + sigma(r, j) * u + i];
            }
            P[s * u + i] = acc;
        }
    }
    return ORACLE_OK;
}

/* O6 rebuild of lost rank k (Eq 2 as "missing = parity XOR survivors", P.481-484,
 * S.330-333; REFT-load step 3 P.545).  For every stripe s and row r != k:
 *   D_k[s(m-1)u + sigma(r,k)u + i] = P_r[s*u + i] XOR
 *                                    XOR_{j not in {r,k}} D_j[s(m-1)u + sigma(r,j)u + i]
 * D[k] and P[k] are ignored (the lost rank's device and host image are gone, Q12).
 * A second loss (lost[] with more than one 1) or m = 1 is unrecoverable (P.460, S.334). */
int oracle_rebuild(uint64_t m, const uint8_t *const *D, const uint8_t *const *P,
                   uint64_t Lstar, uint64_t u, uint64_t k, const uint8_t *lost,
                   uint8_t *Dk)
{
    uint64_t s, i, j, r, nstripes, nlost = 0;
    if (m < 2) return ORACLE_EUNRECOVERABLE;
    if (u == 0 || k >= m || !D || !P || !Dk) return ORACLE_EINVAL;
    if (lost) {
        for (j = 0; j < m; j++) nlost += lost[j] ? 1 : 0;
        if (nlost > 1 || (nlost == 1 && !lost[k])) return ORACLE_EUNRECOVERABLE;
    }
    if (Lstar % ((m - 1) * u)) return ORACLE_EINVAL;
    nstripes = Lstar / ((m - 1) * u);
    for (s = 0; s < nstripes; s++) {
        for (r = 0; r < m; r++) {
            if (r == k) continue;
            for (i = 0; i < u; i++) {
                uint8_t acc = P[r][s * u + i];
                for (j = 0; j < m; j++) {
                    if (j == r || j == k) continue;
                    acc ^= D[j][s * (m - 1) * u + sigma(r, j) * u + i];
                }
                Dk[s * (m - 1) * u + sigma(r, k) * u + i] = acc;
            }
        }
    }
    return ORACLE_OK;
}

/* Seeded synthetic state (SURVEY.md 8(c) "Generator").  This
 * is the oracle's OWN copy of the counter-based generator; the GPU harness has
 * an independent implementation.  Not part of the method.
 *   sm(x): z = x + 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
 *          z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31   (mod 2^64)
 *   base(j, t) = sm(sm(sm(seed) ^ j) ^ t); word w of tensor t = sm(base ^ w),
 *   stored little-endian at byte 8w, tail truncated. */
static uint64_t sm64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t oracle_splitmix64(uint64_t x) { return sm64(x); }

int oracle_fill(uint64_t seed, uint64_t j, uint64_t t, uint64_t byte_begin,
                uint64_t nbytes, uint8_t *out)
{
    uint64_t base = sm64(sm64(sm64(seed) ^ j) ^ t), i;
    if (!out && nbytes) return ORACLE_EINVAL;
    for (i = 0; i < nbytes; i++) {
        uint64_t b = byte_begin + i;
        uint64_t w = sm64(base ^ (b / 8));
        out[i] = (uint8_t)(w >> (8 * (b % 8)));
    }
    return ORACLE_OK;
}

/* ---- ARC and collaborative protection --------------------
 * ARC, "Asynchronous Redundant Copying" (P.456-460): "each member not only saves its own
 * shard to a snapshot but also saves shards from peer members", doubling the volume to
 * 2 W_n/m; placement is the ring of SPEC S.313: member i also holds member (i+1) mod m's
 * image.  Collaborative protection (P.507-508): with ARC and AEC both enabled, "N or
 * fewer node failures" per group (N = 2) are restored.  Reading Q20: the
 * ARC copy in ARC+AEC holds the neighbour's parity row as well as its data, which is
 * what makes every pair of losses recoverable for m >= 3 (an adjacent pair a, a+1
 * would otherwise lose the parity row of a, which covers one unit of every stripe of
 * a+1). */

/* Member holding the ARC copy of member x's image: (x - 1) mod m. */
uint64_t oracle_arc_holder(uint64_t m, uint64_t x) { return (x + m - 1) % m; }

/* ARC copy held by member i: the image of member (i+1) mod m, byte for byte. */
int oracle_arc_copy(uint64_t m, const uint8_t *const *D, uint64_t Lstar, uint64_t i, uint8_t *out)
{
    uint64_t b, src;
    if (m < 2 || i >= m || !D || (!out && Lstar)) return ORACLE_EINVAL;
    src = (i + 1) % m;
    for (b = 0; b < Lstar; b++) out[b] = D[src][b];
    return ORACLE_OK;
}

/* REFT-load step 3 (P.545) for up to two losses.  scheme: 1 = AEC, 2 = ARC, 3 = ARC+AEC.
 * Inputs per member j: D[j] data image (L* bytes), P[j] parity row (L* /(m-1) bytes,
 * AEC schemes), MD[j] / MP[j] the ARC copy of member j+1's data / parity held by j.
 * Entries of lost members are never read.  lost[j] != 0 marks the losses.
 * Outputs, for every lost x: outD[x] (and outP[x] for AEC schemes).
 *   1. every lost x whose holder h = x-1 survived takes D_x = MD[h] (and P_x = MP[h]);
 *   2. if exactly one loss x remains and the scheme has AEC, D_x follows O6 from the
 *      other members' data and parity (restored ones included) and P_x follows O4;
 *   3. anything else is unrecoverable. */
int oracle_recover(uint64_t m, uint64_t scheme, const uint8_t *lost, const uint8_t *const *D,
                   const uint8_t *const *P, const uint8_t *const *MD, const uint8_t *const *MP,
                   uint64_t Lstar, uint64_t u, uint8_t *const *outD, uint8_t *const *outP)
{
    uint64_t j, b, nlost = 0, pbytes, left = 0, x = 0;
    int arc = scheme == 2 || scheme == 3, aec = scheme == 1 || scheme == 3;
    const uint8_t *Dv[8], *Pv[8];
    uint8_t restored[8] = {0};
    if (m < 2 || m > 8 || !lost || !D || !outD || (!arc && !aec)) return m < 2 ? ORACLE_EUNRECOVERABLE : ORACLE_EINVAL;
    if (aec && (u == 0 || Lstar % ((m - 1) * u))) return ORACLE_EINVAL;
    pbytes = Lstar / (m - 1);
    for (j = 0; j < m; j++) nlost += lost[j] ? 1 : 0;
    if (nlost > 2) return ORACLE_EUNRECOVERABLE;
    for (j = 0; j < m; j++) {
        Dv[j] = lost[j] ? 0 : D[j];
        Pv[j] = (lost[j] || !aec) ? 0 : P[j];
    }
    if (arc) {                                   /* step 1 */
        for (j = 0; j < m; j++) {
            uint64_t h = oracle_arc_holder(m, j);
            if (!lost[j] || lost[h]) continue;
            for (b = 0; b < Lstar; b++) outD[j][b] = MD[h][b];
            if (aec) for (b = 0; b < pbytes; b++) outP[j][b] = MP[h][b];
            Dv[j] = outD[j];
            if (aec) Pv[j] = outP[j];
            restored[j] = 1;
        }
    }
    for (j = 0; j < m; j++)
        if (lost[j] && !restored[j]) { left++; x = j; }
    if (left == 0) return ORACLE_OK;
    if (left > 1 || !aec) return ORACLE_EUNRECOVERABLE;
    {                                            /* step 2 */
        int rc = oracle_rebuild(m, Dv, Pv, Lstar, u, x, 0, outD[x]);
        if (rc) return rc;
        Dv[x] = outD[x];
        return oracle_encode(m, Dv, Lstar, u, x, outP[x]);
    }
}

/* ---- AOR, Asynchronous Optimizer Recomputing --------------
 * P.494-505: under ZeRO-1 the optimizer shard of member i has no inherent redundancy,
 * but "model parameters and gradients remain complete on each member"; each member
 * keeps, in host memory, a replica of a peer's optimizer shard and updates it from the
 * gradient of that shard with Eq 4 (P.502-504):
 *     W_opt,shard^(t+1) = W_opt,shard^(t) - eta * grad W_model,shard^(t).
 * Readings: Q22 -- fp32, index order, the product eta*g rounded to fp32
 * before the subtraction (no fused multiply-add; SPEC S.381 "32-bit, sequential, fixed
 * order"); a bf16 gradient is widened exactly to fp32 first.  Q23 -- ring placement as
 * ARC: member i holds the replica of member (i+1) mod m (holder of x = (x-1) mod m). */

/* One Eq 4 step of one replica: w[i] = w[i] - (eta * g[i]) for i = 0..n-1.
 * grad_dtype: 3 = fp32 (g is float[n]), 1 = bf16 (g is uint16[n], bits << 16). */
int oracle_aor_update(uint64_t n, float *w, const void *grad, uint64_t grad_dtype, float eta)
{
    uint64_t i;
    if (n && (!w || !grad)) return ORACLE_EINVAL;
    if (grad_dtype != 3 && grad_dtype != 1) return ORACLE_EINVAL;
    for (i = 0; i < n; i++) {
        float g, prod;
        if (grad_dtype == 3) {
            g = ((const float *)grad)[i];
        } else {
            union { uint32_t u; float f; } cv;
            cv.u = (uint32_t)((const uint16_t *)grad)[i] << 16;
            g = cv.f;
        }
        prod = eta * g;          /* rounded to fp32 (C99, FLT_EVAL_METHOD 0 on x86-64) */
        w[i] = w[i] - prod;
    }
    return ORACLE_OK;
}

/* AOR recovery ("the system retrieves optimizer parameters from host memory with
 * redundant parameters", P.505).  Per member j: master[j] = its optimizer shard
 * (n[j] floats), replica[j] = the replica it holds of member (j+1) mod m (n[(j+1)%m]
 * floats).  Lost members lost both.  Steps:
 *   1. every lost x takes master[x] = replica[holder(x)]; a lost holder -> unrecoverable;
 *   2. every lost x re-creates its replica: replica[x] = master[(x+1) mod m].
 * Nothing is written when the losses are unrecoverable (m = 1 included). */
int oracle_aor_recover(uint64_t m, const uint8_t *lost, float *const *master,
                       float *const *replica, const uint64_t *n)
{
    uint64_t x, i;
    if (m < 1 || m > 8 || !lost || !master || !replica || !n) return ORACLE_EINVAL;
    for (x = 0; x < m; x++)
        if (lost[x] && (m == 1 || lost[oracle_arc_holder(m, x)])) return ORACLE_EUNRECOVERABLE;
    for (x = 0; x < m; x++) {                    /* step 1 */
        if (!lost[x]) continue;
        for (i = 0; i < n[x]; i++) master[x][i] = replica[oracle_arc_holder(m, x)][i];
    }
    for (x = 0; x < m; x++) {                    /* step 2 */
        uint64_t o = (x + 1) % m;
        if (!lost[x]) continue;
        for (i = 0; i < n[o]; i++) replica[x][i] = master[o][i];
    }
    return ORACLE_OK;
}
