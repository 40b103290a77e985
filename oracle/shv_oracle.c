/*
 * shv_oracle.c — plain CPU oracle for the ShoveRand hot path. TEST
 * INFRASTRUCTURE ONLY (see shv_oracle.h): only tests/, smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product never does.
 *
 * Everything here is the textbook definition written out, deliberately in a
 * different formulation from the GPU path:
 *   - MRG32k3a uses L'Ecuyer's signed form  p = a*x - b*y  reduced with C's
 *     '%' (the GPU uses an unsigned rearrangement with 2^32-c folds);
 *   - jumps are generic 3x3 matrix powers with 128-bit accumulation and '%'
 *     (the GPU uses host-built per-bit tables and folded mat-vecs);
 *   - stream positions are (A^(2^127))^g (A^(2^76))^u A^o built by repeated
 *     squaring of A (no per-bit tables);
 *   - Philox serves lanes through the SPEC's next_word buffer, one draw at a
 *     time (the GPU computes whole counter blocks per store).
 * Compiled with -O2 -ffp-contract=off. No SIMD, no lookup tables.
 */
#include "shv_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* MRG32k3a parameters, [LEcuyer1999] Table II (cited at P L84, L255):
 *   x1,n = (1403580 x1,n-2 - 810728 x1,n-3) mod m1
 *   x2,n = (527612 x2,n-1 - 1370589 x2,n-3) mod m2
 *   z_n  = (x1,n - x2,n) mod m1, returned as m1 when it is 0 (R2). */
static const int64_t m1 = 4294967087LL; /* 2^32 - 209   */
static const int64_t m2 = 4294944443LL; /* 2^32 - 22853 */
static const int64_t a12 = 1403580LL;
static const int64_t a13n = 810728LL;
static const int64_t a21 = 527612LL;
static const int64_t a23n = 1370589LL;

/* [LEcuyer1999]'s normalisation constant 1/(m1+1) as printed in his code
 * ("#define norm 2.328306549295727688e-10"); R7. */
static const double mrg_norm = 2.328306549295727688e-10;

/* Philox4x32 constants, [Salmon.etal.2011] §3.3 / Random123 (P L327). */
static const uint32_t PHILOX_M0 = 0xD2511F53u;
static const uint32_t PHILOX_M1 = 0xCD9E8D57u;
static const uint32_t PHILOX_W0 = 0x9E3779B9u; /* golden ratio */
static const uint32_t PHILOX_W1 = 0xBB67AE85u; /* sqrt(3) - 1   */

/* ------------------------------------------------------------------------ */
/* MRG32k3a                                                                  */
/* ------------------------------------------------------------------------ */

uint32_t orc_mrg_step(uint32_t s[6])
{
    /* State (x1,n-3, x1,n-2, x1,n-1, x2,n-3, x2,n-2, x2,n-1) = s[0..5] (R1). */
    int64_t p1 = a12 * (int64_t)s[1] - a13n * (int64_t)s[0];
    p1 %= m1;
    if (p1 < 0) p1 += m1;
    int64_t p2 = a21 * (int64_t)s[5] - a23n * (int64_t)s[3];
    p2 %= m2;
    if (p2 < 0) p2 += m2;
    s[0] = s[1]; s[1] = s[2]; s[2] = (uint32_t)p1;
    s[3] = s[4]; s[4] = s[5]; s[5] = (uint32_t)p2;
    /* Combination, [LEcuyer1999]: (p1 - p2) mod m1 with 0 mapped to m1. */
    if (p1 > p2) return (uint32_t)(p1 - p2);
    return (uint32_t)(p1 - p2 + m1);
}

void orc_mrg_matrices(uint64_t A1[9], uint64_t A2[9])
{
    /* Companion matrices acting on the column (x_{n-3}, x_{n-2}, x_{n-1}):
     * the new last entry is the recurrence, the others shift up (R3). */
    const uint64_t a[9] = {0, 1, 0,
                           0, 0, 1,
                           (uint64_t)(m1 - a13n), (uint64_t)a12, 0};
    const uint64_t b[9] = {0, 1, 0,
                           0, 0, 1,
                           (uint64_t)(m2 - a23n), 0, (uint64_t)a21};
    memcpy(A1, a, sizeof a);
    memcpy(A2, b, sizeof b);
}

void orc_mat_mul(const uint64_t A[9], const uint64_t B[9], uint64_t m, uint64_t C[9])
{
    uint64_t T[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            u128 acc = 0;
            for (int k = 0; k < 3; ++k) acc += (u128)A[3 * r + k] * B[3 * k + c];
            T[3 * r + c] = (uint64_t)(acc % m);
        }
    memcpy(C, T, sizeof T);
}

void orc_mat_pow(const uint64_t A[9], uint64_t e_lo, uint64_t e_hi, uint64_t m, uint64_t out[9])
{
    u128 e = ((u128)e_hi << 64) | e_lo;
    uint64_t R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    uint64_t P[9];
    memcpy(P, A, sizeof P);
    while (e) {
        if (e & 1) orc_mat_mul(R, P, m, R);
        orc_mat_mul(P, P, m, P);
        e >>= 1;
    }
    memcpy(out, R, sizeof R);
}

static void mat_vec(const uint64_t M[9], const uint32_t v[3], uint64_t m, uint32_t out[3])
{
    uint32_t t[3];
    for (int r = 0; r < 3; ++r) {
        u128 acc = 0;
        for (int k = 0; k < 3; ++k) acc += (u128)M[3 * r + k] * v[k];
        t[r] = (uint32_t)(acc % m);
    }
    memcpy(out, t, sizeof t);
}

void orc_mrg_jump(uint32_t s[6], uint64_t e_lo, uint64_t e_hi)
{
    uint64_t A1[9], A2[9], P1[9], P2[9];
    orc_mrg_matrices(A1, A2);
    orc_mat_pow(A1, e_lo, e_hi, (uint64_t)m1, P1);
    orc_mat_pow(A2, e_lo, e_hi, (uint64_t)m2, P2);
    mat_vec(P1, s, (uint64_t)m1, s);
    mat_vec(P2, s + 3, (uint64_t)m2, s + 3);
}

/* A^(2^k) by k squarings. */
static void mat_pow2k(const uint64_t A[9], int k, uint64_t m, uint64_t out[9])
{
    uint64_t P[9];
    memcpy(P, A, sizeof P);
    for (int i = 0; i < k; ++i) orc_mat_mul(P, P, m, P);
    memcpy(out, P, sizeof P);
}

void orc_mrg_position(const uint32_t seed[6], uint64_t g, uint64_t u,
                      uint64_t o_lo, uint64_t o_hi, uint32_t out[6])
{
    /* Position g*2^127 + u*2^76 + o (P L264-268: 2^64 streams of 2^127,
     * substreams of 2^76). The exponent can reach 2^191, so it is applied as
     * three matrix powers rather than one (R4). */
    uint64_t A[2][9], S127[9], S76[9], Pg[9], Pu[9], Po[9], M[9];
    const uint64_t mod[2] = {(uint64_t)m1, (uint64_t)m2};
    orc_mrg_matrices(A[0], A[1]);
    for (int c = 0; c < 2; ++c) {
        mat_pow2k(A[c], 127, mod[c], S127);
        mat_pow2k(A[c], 76, mod[c], S76);
        orc_mat_pow(S127, g, 0, mod[c], Pg);
        orc_mat_pow(S76, u, 0, mod[c], Pu);
        orc_mat_pow(A[c], o_lo, o_hi, mod[c], Po);
        orc_mat_mul(Pg, Pu, mod[c], M);
        orc_mat_mul(M, Po, mod[c], M);
        mat_vec(M, seed + 3 * c, mod[c], out + 3 * c);
    }
}

/* ------------------------------------------------------------------------ */
/* Philox4x32                                                                */
/* ------------------------------------------------------------------------ */

static void mulhilo(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo)
{
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

void orc_philox_block(const uint32_t ctr[4], const uint32_t key[2], int rounds, uint32_t out[4])
{
    /* [Salmon.etal.2011] Philox S-P network, N=4, W=32:
     *   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2
     *   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
     * with the Weyl key bump k += (W0, W1) between rounds (R5). */
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < rounds; ++r) {
        if (r > 0) {
            k0 += PHILOX_W0;
            k1 += PHILOX_W1;
        }
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo(PHILOX_M0, c[0], &hi0, &lo0);
        mulhilo(PHILOX_M1, c[2], &hi1, &lo1);
        uint32_t n0 = hi1 ^ c[1] ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c[3] ^ k1;
        uint32_t n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    memcpy(out, c, sizeof c);
}

/* ------------------------------------------------------------------------ */
/* Threefry4x64 ([Salmon.etal.2011] §3.2: Threefish-256 with a 20-round ARX  */
/* schedule, key injection every 4 rounds, no tweak)                        */
/* ------------------------------------------------------------------------ */

static uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

void orc_threefry4x64_block(const uint64_t ctr[4], const uint64_t key[4], int rounds, uint64_t out[4])
{
    /* Threefish-256 rotation constants and the key-schedule parity word. */
    static const int R[8][2] = {{14, 16}, {52, 57}, {23, 40}, {5, 37},
                                {25, 33}, {46, 12}, {58, 22}, {32, 32}};
    uint64_t ks[5];
    ks[4] = 0x1BD11BDAA9FC1A22ull;
    for (int i = 0; i < 4; ++i) {
        ks[i] = key[i];
        ks[4] ^= key[i];
    }
    uint64_t x[4];
    for (int i = 0; i < 4; ++i) x[i] = ctr[i] + ks[i];
    for (int r = 0; r < rounds; ++r) {
        if (r % 2 == 0) { /* mix (0,1), (2,3) */
            x[0] += x[1]; x[1] = rotl64(x[1], R[r % 8][0]) ^ x[0];
            x[2] += x[3]; x[3] = rotl64(x[3], R[r % 8][1]) ^ x[2];
        } else { /* permuted: mix (0,3), (2,1) */
            x[0] += x[3]; x[3] = rotl64(x[3], R[r % 8][0]) ^ x[0];
            x[2] += x[1]; x[1] = rotl64(x[1], R[r % 8][1]) ^ x[2];
        }
        if (r % 4 == 3) { /* key injection s = (r+1)/4 */
            const uint64_t inj = (uint64_t)(r + 1) / 4;
            for (int i = 0; i < 4; ++i) x[i] += ks[(inj + i) % 5];
            x[3] += inj;
        }
    }
    memcpy(out, x, sizeof x);
}

/* ------------------------------------------------------------------------ */
/* TinyMT32 ([Saito2011]: tinymt32.h/.c of the authors' distribution)       */
/* ------------------------------------------------------------------------ */

#define TINYMT32_MASK 0x7fffffffu
#define TINYMT32_SH0 1
#define TINYMT32_SH1 10
#define TINYMT32_SH8 8

void orc_tinymt32_next_state(orc_tinymt32* t)
{
    uint32_t x, y;
    y = t->st[3];
    x = (t->st[0] & TINYMT32_MASK) ^ t->st[1] ^ t->st[2];
    x ^= (x << TINYMT32_SH0);
    y ^= (y >> TINYMT32_SH0) ^ x;
    t->st[0] = t->st[1];
    t->st[1] = t->st[2];
    t->st[2] = x ^ (y << TINYMT32_SH1);
    t->st[3] = y;
    t->st[1] ^= (uint32_t)(-(int32_t)(y & 1)) & t->mat1;
    t->st[2] ^= (uint32_t)(-(int32_t)(y & 1)) & t->mat2;
}

uint32_t orc_tinymt32_temper(const orc_tinymt32* t)
{
    uint32_t t0, t1;
    t0 = t->st[3];
    t1 = t->st[0] + (t->st[2] >> TINYMT32_SH8);
    t0 ^= t1;
    t0 ^= (uint32_t)(-(int32_t)(t1 & 1)) & t->tmat;
    return t0;
}

uint32_t orc_tinymt32_generate(orc_tinymt32* t)
{
    orc_tinymt32_next_state(t);
    return orc_tinymt32_temper(t);
}

void orc_tinymt32_init(orc_tinymt32* t, uint32_t mat1, uint32_t mat2, uint32_t tmat, uint32_t seed)
{
    t->mat1 = mat1;
    t->mat2 = mat2;
    t->tmat = tmat;
    t->st[0] = seed;
    t->st[1] = mat1;
    t->st[2] = mat2;
    t->st[3] = tmat;
    for (int i = 1; i < 8; i++)
        t->st[i & 3] ^= (uint32_t)i + 1812433253u * (t->st[(i - 1) & 3] ^ (t->st[(i - 1) & 3] >> 30));
    /* period certification: the 127 significant bits must not all be zero */
    if ((t->st[0] & TINYMT32_MASK) == 0 && t->st[1] == 0 && t->st[2] == 0 && t->st[3] == 0) {
        t->st[0] = 'T';
        t->st[1] = 'I';
        t->st[2] = 'N';
        t->st[3] = 'Y';
    }
    for (int i = 0; i < 8; i++) orc_tinymt32_next_state(t);
}

/* 128x128 matrices over GF(2): row r is bits r of the image; M[r][w] holds
 * 32 columns. Column c of T = next_state(e_c), so y = T x is the XOR of the
 * columns selected by the bits of x. Stored column-major: col[c][4]. */
typedef struct { uint32_t col[128][4]; } gf2mat;

static void gf2_apply(const gf2mat* M, const uint32_t x[4], uint32_t y[4])
{
    uint32_t r[4] = {0, 0, 0, 0};
    for (int c = 0; c < 128; ++c)
        if ((x[c >> 5] >> (c & 31)) & 1)
            for (int w = 0; w < 4; ++w) r[w] ^= M->col[c][w];
    memcpy(y, r, sizeof r);
}

static void gf2_mul(const gf2mat* A, const gf2mat* B, gf2mat* C) /* C = A B */
{
    gf2mat T;
    for (int c = 0; c < 128; ++c) gf2_apply(A, B->col[c], T.col[c]);
    *C = T;
}

/* R = T^e for the transition T of t's parameter set (square-and-multiply). */
static void tinymt32_pow(const orc_tinymt32* t, u128 e, gf2mat* out)
{
    gf2mat P, R;
    memset(&R, 0, sizeof R);
    for (int c = 0; c < 128; ++c) R.col[c][c >> 5] = 1u << (c & 31); /* identity */
    for (int c = 0; c < 128; ++c) { /* P = T */
        orc_tinymt32 u = *t;
        memset(u.st, 0, sizeof u.st);
        u.st[c >> 5] = 1u << (c & 31);
        orc_tinymt32_next_state(&u);
        memcpy(P.col[c], u.st, sizeof u.st);
    }
    while (e) {
        if (e & 1) gf2_mul(&P, &R, &R);
        gf2_mul(&P, &P, &P);
        e >>= 1;
    }
    *out = R;
}

void orc_tinymt32_jump(orc_tinymt32* t, uint64_t e_lo, uint64_t e_hi)
{
    gf2mat P, R;
    memset(&R, 0, sizeof R);
    for (int c = 0; c < 128; ++c) R.col[c][c >> 5] = 1u << (c & 31); /* identity */
    for (int c = 0; c < 128; ++c) { /* P = T */
        orc_tinymt32 u = *t;
        memset(u.st, 0, sizeof u.st);
        u.st[c >> 5] = 1u << (c & 31);
        orc_tinymt32_next_state(&u);
        memcpy(P.col[c], u.st, sizeof u.st);
    }
    u128 e = ((u128)e_hi << 64) | e_lo;
    while (e) {
        if (e & 1) gf2_mul(&P, &R, &R);
        gf2_mul(&P, &P, &P);
        e >>= 1;
    }
    gf2_apply(&R, t->st, t->st);
}

/* ------------------------------------------------------------------------ */
/* MTGP32 ([Saito.Matsumoto2012]; P L74-76, L133-136), MEXP 11213            */
/* ------------------------------------------------------------------------ */

void orc_mtgp32_init(orc_mtgp32* m, const orc_mtgp32_params* p, uint32_t seed)
{
    const int n = ORC_MTGP32_N; /* mexp / 32 + 1 */
    m->p = *p;
    m->idx = 0;
    const uint32_t hidden = p->tbl[4] ^ (p->tbl[8] << 16);
    uint32_t fill = hidden;
    fill += fill >> 16;
    fill += fill >> 8;
    fill &= 0xffu;
    for (int i = 0; i < n; ++i) m->x[i] = fill * 0x01010101u; /* every byte = fill */
    m->x[0] = seed;
    m->x[1] = hidden;
    for (int i = 1; i < n; ++i)
        m->x[i] ^= 1812433253u * (m->x[i - 1] ^ (m->x[i - 1] >> 30)) + (uint32_t)i;
}

uint32_t orc_mtgp32_generate(orc_mtgp32* m)
{
    const int n = ORC_MTGP32_N;
    const orc_mtgp32_params* p = &m->p;
    const uint32_t x1 = m->x[m->idx];                           /* x_k */
    const uint32_t x2 = m->x[(m->idx + 1) % n];                 /* x_{k+1} */
    uint32_t y = m->x[(m->idx + (int)p->pos) % n];              /* x_{k+pos} */
    const uint32_t t = m->x[(m->idx + (int)p->pos - 1) % n];    /* x_{k+pos-1} */
    /* recursion (para_rec) */
    uint32_t x = (x1 & p->mask) ^ x2;
    x ^= x << p->sh1;
    y = x ^ (y >> p->sh2);
    const uint32_t r = y ^ p->tbl[y & 0x0f];
    m->x[m->idx] = r; /* x_{k+N} takes x_k's slot */
    m->idx = (m->idx + 1) % n;
    /* tempering */
    uint32_t u = t;
    u ^= u >> 16;
    u ^= u >> 8;
    return r ^ p->tmp_tbl[u & 0x0f];
}

/* ------------------------------------------------------------------------ */
/* conversions (R7)                                                          */
/* ------------------------------------------------------------------------ */

float orc_to_f32(uint32_t w) { return (float)(w >> 8) * 0x1p-24f; }

double orc_mrg_to_f64(uint32_t z) { return (double)z * mrg_norm; }

double orc_philox_to_f64(uint32_t lo, uint32_t hi)
{
    uint64_t b = ((uint64_t)hi << 32) | lo;
    return (double)(b >> 11) * 0x1p-53;
}

/* ------------------------------------------------------------------------ */
/* streams (P L387-399: the per-PE object and next())                        */
/* ------------------------------------------------------------------------ */

static int seed_words_mrg(const uint32_t* seed, int nseed, uint32_t s[6])
{
    if (nseed == 1) {
        for (int k = 0; k < 6; ++k) s[k] = seed[0];
    } else if (nseed == 6) {
        for (int k = 0; k < 6; ++k) s[k] = seed[k];
    } else {
        return -1;
    }
    /* S L114-119: residues in range, neither triple all zero. */
    for (int k = 0; k < 3; ++k)
        if ((int64_t)s[k] >= m1 || (int64_t)s[3 + k] >= m2) return -1;
    if (!(s[0] | s[1] | s[2]) || !(s[3] | s[4] | s[5])) return -1;
    return 0;
}

int orc_stream_open(orc_stream* st, int gen, const uint32_t* seed, int nseed,
                    uint64_t first, uint64_t i, int spacing,
                    uint64_t off_lo, uint64_t off_hi)
{
    memset(st, 0, sizeof *st);
    st->gen = gen;
    if (gen == ORC_MRG32K3A) {
        uint32_t base[6];
        if (seed_words_mrg(seed, nseed, base)) return -1;
        /* Handle-stream i is stream first+i (STREAM) or substream first+i of
         * stream 0 (SUBSTREAM) (R4). */
        uint64_t g = 0, u = 0;
        if (spacing == ORC_SPACING_STREAM) g = first + i;
        else if (spacing == ORC_SPACING_SUBSTREAM) u = first + i;
        else return -1;
        orc_mrg_position(base, g, u, off_lo, off_hi, st->s);
        return 0;
    }
    if (gen == ORC_TINYMT32) {
        /* seed = {seed, group_size, n_params, params...} (R15) */
        if (nseed < 6 || spacing != ORC_SPACING_STREAM) return -1;
        const uint32_t gs = seed[1], np = seed[2];
        if (gs == 0 || (uint64_t)nseed != 3 + 3ull * np) return -1;
        const uint64_t g = first + i, group = g / gs, slice = g % gs;
        if (group >= np) return -1; /* one parameter set per group */
        const uint32_t* p = seed + 3 + 3 * group;
        orc_tinymt32_init(&st->tm, p[0], p[1], p[2], seed[0]);
        /* slice start: 2^64 * slice draws (u128 exponent: slice < 2^64) */
        orc_tinymt32_jump(&st->tm, 0, slice);
        orc_tinymt32_jump(&st->tm, off_lo, off_hi);
        return 0;
    }
    if (gen == ORC_MTGP32) {
        /* seed = {seed_lo, seed_hi, n_params, 36 words per set} (R18) */
        if (nseed < 3 || spacing != ORC_SPACING_STREAM || off_hi) return -1;
        const uint32_t np = seed[2];
        if ((uint64_t)nseed != 3 + 36ull * np) return -1;
        const uint64_t g = first + i;
        if (g >= np) return -1; /* one parameter set per state */
        const uint32_t* w = seed + 3 + 36 * g;
        orc_mtgp32_params p;
        p.pos = w[0];
        p.sh1 = w[1];
        p.sh2 = w[2];
        p.mask = w[3];
        for (int k = 0; k < 16; ++k) {
            p.tbl[k] = w[4 + k];
            p.tmp_tbl[k] = w[20 + k];
        }
        if (p.pos < 2 || p.pos >= ORC_MTGP32_N || p.sh1 > 31 || p.sh2 > 31) return -1;
        const uint64_t s64 = (uint64_t)seed[0] | ((uint64_t)seed[1] << 32);
        orc_mtgp32_init(&st->mt, &p, (uint32_t)(s64 ^ (s64 >> 32)) + (uint32_t)g + 1u);
        for (uint64_t k = 0; k < off_lo; ++k) (void)orc_mtgp32_generate(&st->mt);
        return 0;
    }
    if (gen == ORC_THREEFRY4X64_20) {
        /* R16: key = (s0 | s1<<32, s2 | s3<<32, 0, 0) from 1..4 seed words;
         * stream g -> ctr = (blk, g, 0, 0); draw d -> word d & 7 of block
         * d >> 3, words = (lo, hi) of lanes 0..3. */
        if (nseed < 1 || nseed > 4 || spacing != ORC_SPACING_STREAM) return -1;
        if (off_hi >> 3) return -1; /* a stream holds 2^67 draws */
        uint32_t w[4] = {0, 0, 0, 0};
        for (int k = 0; k < nseed; ++k) w[k] = seed[k];
        st->tkey[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
        st->tkey[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
        st->tkey[2] = st->tkey[3] = 0;
        st->g = first + i;
        u128 d = ((u128)off_hi << 64) | off_lo;
        st->blk = (uint64_t)(d >> 3);
        st->tpos = 8;
        int word = (int)(d & 7);
        if (word) {
            (void)orc_stream_next(st); /* fill the buffer at block d>>3 */
            st->tpos = word;
        }
        return 0;
    }
    if (gen == ORC_PHILOX4X32_10) {
        if (off_hi >> 2) return -1; /* a stream holds 2^66 draws (R6) */
        if (spacing == ORC_SPACING_STREAM) {
            if (nseed != 1 && nseed != 2) return -1;
            st->key[0] = seed[0];
            st->key[1] = nseed == 2 ? seed[1] : 0;
            st->g = first + i;
        } else if (spacing == ORC_SPACING_KEYED) {
            /* Parameterization by key (P L331-334: "a single key that can be
             * set at runtime according to each thread's unique identifier";
             * S L249-257): key0 = stream id, key1 = experiment tag = seed[0];
             * counter = (blk_lo, blk_hi, 0, 0). Ids beyond 2^32 exhaust the
             * key word (S L253). */
            if (nseed != 1) return -1;
            if (first + i > 0xFFFFFFFFull || first + i < first) return -1;
            st->key[0] = (uint32_t)(first + i);
            st->key[1] = seed[0];
            st->g = 0;
        } else {
            return -1;
        }
        u128 d = ((u128)off_hi << 64) | off_lo;
        st->blk = (uint64_t)(d >> 2);
        st->buf_pos = 4;
        int lane = (int)(d & 3);
        if (lane) {
            (void)orc_stream_next(st); /* fill the buffer at block d>>2 */
            st->buf_pos = lane;
        }
        return 0;
    }
    return -1;
}

int orc_stream_open_leapfrog(orc_stream* st, int gen, const uint32_t* seed, int nseed,
                             uint64_t players, uint64_t player, uint64_t off_lo, uint64_t off_hi)
{
    if (players == 0 || player >= players) return -1;
    const u128 off = ((u128)off_hi << 64) | off_lo;
    /* d0 = player + K*off, the first base draw this player receives */
    if (off > (~(u128)0 - player) / players) return -1;
    const u128 d0 = (u128)player + (u128)players * off;
    if (gen == ORC_MRG32K3A) {
        if (orc_stream_open(st, gen, seed, nseed, 0, 0, ORC_SPACING_STREAM, (uint64_t)d0,
                            (uint64_t)(d0 >> 64)))
            return -1;
        uint64_t A1[9], A2[9];
        orc_mrg_matrices(A1, A2);
        orc_mat_pow(A1, players - 1, 0, (uint64_t)m1, st->leapA1);
        orc_mat_pow(A2, players - 1, 0, (uint64_t)m2, st->leapA2);
    } else if (gen == ORC_TINYMT32) {
        /* R19: the base sequence is TinyMT32 init(params, seed) with seed =
         * {seed, mat1, mat2, tmat}; the player's state is the base state after
         * d0 draws (T^d0, S L355 jump = iterate); each draw then discards K-1
         * base draws by stepping (K <= 65, SPEC's per-PE stride-k stepping,
         * S L424) or by the matrix T^(K-1) (larger K). */
        if (nseed != 4) return -1;
        memset(st, 0, sizeof *st);
        st->gen = gen;
        orc_tinymt32_init(&st->tm, seed[1], seed[2], seed[3], seed[0]);
        orc_tinymt32_jump(&st->tm, (uint64_t)d0, (uint64_t)(d0 >> 64));
        if (players - 1 > 64) {
            gf2mat M;
            tinymt32_pow(&st->tm, (u128)(players - 1), &M);
            memcpy(st->leapT, M.col, sizeof st->leapT);
        }
    } else if (gen == ORC_PHILOX4X32_10 || gen == ORC_THREEFRY4X64_20) {
        if (orc_stream_open(st, gen, seed, nseed, 0, 0, ORC_SPACING_STREAM, 0, 0)) return -1;
        if (d0 >= ((u128)1 << (gen == ORC_PHILOX4X32_10 ? 66 : 67))) return -1;
        st->pos_lo = (uint64_t)d0;
        st->pos_hi = (uint64_t)(d0 >> 64);
    } else {
        return -1;
    }
    st->leap = players;
    return 0;
}

/* Draw at base index d of counter stream 0 (Leap Frog, R17). */
static uint32_t counter_word(const orc_stream* st, u128 d)
{
    if (st->gen == ORC_THREEFRY4X64_20) {
        const uint64_t ctr[4] = {(uint64_t)(d >> 3), 0, 0, 0};
        uint64_t out[4];
        orc_threefry4x64_block(ctr, st->tkey, 20, out);
        const uint64_t lane = out[(d & 7) >> 1];
        return (d & 1) ? (uint32_t)(lane >> 32) : (uint32_t)lane;
    }
    const uint64_t b = (uint64_t)(d >> 2);
    const uint32_t ctr[4] = {(uint32_t)b, (uint32_t)(b >> 32), 0, 0};
    uint32_t out[4];
    orc_philox_block(ctr, st->key, 10, out);
    return out[d & 3];
}

uint32_t orc_stream_next(orc_stream* st)
{
    if (st->leap) {
        /* Leap Frog: serve the next base draw, then skip K-1 base draws. */
        if (st->gen == ORC_TINYMT32) {
            const uint32_t w = orc_tinymt32_generate(&st->tm);
            if (st->leap - 1 > 64) {
                gf2mat M;
                memcpy(M.col, st->leapT, sizeof M.col);
                gf2_apply(&M, st->tm.st, st->tm.st);
            } else {
                for (uint64_t k = 1; k < st->leap; ++k) orc_tinymt32_next_state(&st->tm);
            }
            return w;
        }
        if (st->gen == ORC_MRG32K3A) {
            const uint32_t z = orc_mrg_step(st->s);
            uint32_t a[3], b[3];
            mat_vec(st->leapA1, st->s, (uint64_t)m1, a);
            mat_vec(st->leapA2, st->s + 3, (uint64_t)m2, b);
            memcpy(st->s, a, sizeof a);
            memcpy(st->s + 3, b, sizeof b);
            return z;
        }
        const u128 d = ((u128)st->pos_hi << 64) | st->pos_lo;
        const uint32_t w = counter_word(st, d);
        const u128 nd = d + st->leap;
        st->pos_lo = (uint64_t)nd;
        st->pos_hi = (uint64_t)(nd >> 64);
        return w;
    }
    if (st->gen == ORC_MRG32K3A) return orc_mrg_step(st->s);
    if (st->gen == ORC_TINYMT32) return orc_tinymt32_generate(&st->tm);
    if (st->gen == ORC_MTGP32) return orc_mtgp32_generate(&st->mt);
    if (st->gen == ORC_THREEFRY4X64_20) {
        if (st->tpos == 8) {
            const uint64_t ctr[4] = {st->blk, st->g, 0, 0};
            uint64_t out[4];
            orc_threefry4x64_block(ctr, st->tkey, 20, out);
            for (int l = 0; l < 4; ++l) {
                st->tbuf[2 * l] = (uint32_t)out[l];
                st->tbuf[2 * l + 1] = (uint32_t)(out[l] >> 32);
            }
            st->blk += 1;
            st->tpos = 0;
        }
        return st->tbuf[st->tpos++];
    }
    /* SPEC next_word (S L258-266): serve x, y, z, w of the current block,
     * then evaluate the next counter. Counter = (blk_lo, blk_hi, g_lo, g_hi),
     * key = (seed0, seed1) (R6). */
    if (st->buf_pos == 4) {
        uint32_t ctr[4] = {(uint32_t)st->blk, (uint32_t)(st->blk >> 32),
                           (uint32_t)st->g, (uint32_t)(st->g >> 32)};
        orc_philox_block(ctr, st->key, 10, st->buf);
        st->blk += 1;
        st->buf_pos = 0;
    }
    return st->buf[st->buf_pos++];
}

/* ------------------------------------------------------------------------ */
/* bulk rows and Monte Carlo, split over threads by contiguous stream ranges */
/* ------------------------------------------------------------------------ */

typedef struct {
    int gen, nseed, spacing, kind, mc;
    uint64_t players;                  /* Leap Frog: K (spacing LEAPFROG) */
    const uint32_t* seed;
    uint64_t first, off_lo, off_hi, n; /* n = values per row, or samples */
    const uint64_t* idx;               /* NULL: row r is stream r */
    uint64_t r0, r1;                   /* rows [r0, r1) */
    void* out;
    uint64_t* counts;
    uint64_t total;
    int err;
} job_t;

static void* run_job(void* arg)
{
    job_t* jb = (job_t*)arg;
    for (uint64_t r = jb->r0; r < jb->r1; ++r) {
        uint64_t i = jb->idx ? jb->idx[r] : r;
        orc_stream st;
        const int bad = jb->spacing == ORC_SPACING_LEAPFROG
                            ? orc_stream_open_leapfrog(&st, jb->gen, jb->seed, jb->nseed, jb->players,
                                                       jb->first + i, jb->off_lo, jb->off_hi)
                            : orc_stream_open(&st, jb->gen, jb->seed, jb->nseed, jb->first, i,
                                              jb->spacing, jb->off_lo, jb->off_hi);
        if (bad) {
            jb->err = 1;
            return NULL;
        }
        if (jb->mc) {
            /* Dartboard (S L529-537): x = w>>8, y = w'>>8 as 24-bit lattice
             * points; x^2 + y^2 < 1 on the f32 values iff X^2+Y^2 < 2^48 (R9). */
            uint64_t hits = 0;
            for (uint64_t k = 0; k < jb->n; ++k) {
                uint64_t X = orc_stream_next(&st) >> 8;
                uint64_t Y = orc_stream_next(&st) >> 8;
                if (X * X + Y * Y < ((uint64_t)1 << 48)) ++hits;
            }
            if (jb->counts) jb->counts[r] = hits;
            jb->total += hits;
            continue;
        }
        for (uint64_t j = 0; j < jb->n; ++j) {
            uint64_t at = r * jb->n + j;
            if (jb->kind == ORC_U32) {
                ((uint32_t*)jb->out)[at] = orc_stream_next(&st);
            } else if (jb->kind == ORC_F32) {
                ((float*)jb->out)[at] = orc_to_f32(orc_stream_next(&st));
            } else if (jb->gen == ORC_MRG32K3A) {
                ((double*)jb->out)[at] = orc_mrg_to_f64(orc_stream_next(&st));
            } else { /* Philox, TinyMT32, MTGP32: 53 bits from two consecutive words (R7) */
                uint32_t lo = orc_stream_next(&st);
                uint32_t hi = orc_stream_next(&st);
                ((double*)jb->out)[at] = orc_philox_to_f64(lo, hi);
            }
        }
    }
    return NULL;
}

static int run_jobs(job_t proto, uint64_t rows, int nthreads, uint64_t* total)
{
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > rows) nthreads = rows ? (int)rows : 1;
    job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) {
        free(jobs);
        free(th);
        return -1;
    }
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = proto;
        jobs[t].r0 = rows * (uint64_t)t / (uint64_t)nthreads;
        jobs[t].r1 = rows * (uint64_t)(t + 1) / (uint64_t)nthreads;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, run_job, &jobs[t]);
    run_job(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    int err = 0;
    uint64_t sum = 0;
    for (int t = 0; t < nthreads; ++t) {
        err |= jobs[t].err;
        sum += jobs[t].total;
    }
    free(jobs);
    free(th);
    if (total) *total = sum;
    return err ? -1 : 0;
}

static job_t make_job(int gen, const uint32_t* seed, int nseed, uint64_t first, int spacing,
                      uint64_t off_lo, uint64_t off_hi, uint64_t n, int kind,
                      const uint64_t* idx, void* out, uint64_t* counts, int mc)
{
    job_t j;
    memset(&j, 0, sizeof j);
    j.gen = gen; j.seed = seed; j.nseed = nseed; j.first = first; j.spacing = spacing;
    j.off_lo = off_lo; j.off_hi = off_hi; j.n = n; j.kind = kind; j.idx = idx;
    j.out = out; j.counts = counts; j.mc = mc;
    return j;
}

int orc_generate(int gen, const uint32_t* seed, int nseed, uint64_t first,
                 uint64_t n_streams, int spacing, uint64_t off_lo, uint64_t off_hi,
                 uint64_t n, int kind, void* out, int nthreads)
{
    job_t p = make_job(gen, seed, nseed, first, spacing, off_lo, off_hi, n, kind, NULL, out, NULL, 0);
    return run_jobs(p, n_streams, nthreads, NULL);
}

int orc_generate_list(int gen, const uint32_t* seed, int nseed, uint64_t first,
                      const uint64_t* idx, uint64_t n_idx, int spacing,
                      uint64_t off_lo, uint64_t off_hi, uint64_t n, int kind,
                      void* out, int nthreads)
{
    job_t p = make_job(gen, seed, nseed, first, spacing, off_lo, off_hi, n, kind, idx, out, NULL, 0);
    return run_jobs(p, n_idx, nthreads, NULL);
}

uint64_t orc_mc_count(int gen, const uint32_t* seed, int nseed, uint64_t first,
                      uint64_t n_streams, int spacing, uint64_t off_lo, uint64_t off_hi,
                      uint64_t samples, uint64_t* counts, int nthreads)
{
    uint64_t total = 0;
    job_t p = make_job(gen, seed, nseed, first, spacing, off_lo, off_hi, samples, 0, NULL, NULL, counts, 1);
    if (run_jobs(p, n_streams, nthreads, &total)) return UINT64_MAX;
    return total;
}

uint64_t orc_mc_count_list(int gen, const uint32_t* seed, int nseed, uint64_t first,
                           const uint64_t* idx, uint64_t n_idx, int spacing,
                           uint64_t off_lo, uint64_t off_hi, uint64_t samples,
                           uint64_t* counts, int nthreads)
{
    uint64_t total = 0;
    job_t p = make_job(gen, seed, nseed, first, spacing, off_lo, off_hi, samples, 0, idx, NULL, counts, 1);
    if (run_jobs(p, n_idx, nthreads, &total)) return UINT64_MAX;
    return total;
}

int orc_generate_leapfrog(int gen, const uint32_t* seed, int nseed, uint64_t players, uint64_t first,
                          const uint64_t* idx, uint64_t n_rows, uint64_t off_lo, uint64_t off_hi,
                          uint64_t n, int kind, void* out, int nthreads)
{
    job_t p = make_job(gen, seed, nseed, first, ORC_SPACING_LEAPFROG, off_lo, off_hi, n, kind, idx,
                       out, NULL, 0);
    p.players = players;
    return run_jobs(p, n_rows, nthreads, NULL);
}

uint64_t orc_mc_count_leapfrog(int gen, const uint32_t* seed, int nseed, uint64_t players,
                               uint64_t first, const uint64_t* idx, uint64_t n_rows, uint64_t off_lo,
                               uint64_t off_hi, uint64_t samples, uint64_t* counts, int nthreads)
{
    uint64_t total = 0;
    job_t p = make_job(gen, seed, nseed, first, ORC_SPACING_LEAPFROG, off_lo, off_hi, samples, 0, idx,
                       NULL, counts, 1);
    p.players = players;
    if (run_jobs(p, n_rows, nthreads, &total)) return UINT64_MAX;
    return total;
}
