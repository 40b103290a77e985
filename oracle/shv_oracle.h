/*
 * shv_oracle.h — plain, slow, obviously-correct CPU oracle for the ShoveRand
 * hot path (arXiv 1412.8266). TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path
 * (paper_1412_8266_b200/, include/shv.h) shares no code, header, table or
 * constant generator with this file, and never calls it.
 *
 * Citations: "P Lnn" = /root/reference/PAPER.md line nn, "S Lnn" = SPEC.md
 * line nn. Readings of silent/ambiguous points are listed in DESIGN.md §3
 * (R1..R12) and referenced here by their ID.
 */
#ifndef SHV_ORACLE_H
#define SHV_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_MRG32K3A = 1, ORC_PHILOX4X32_10 = 2, ORC_TINYMT32 = 3, ORC_THREEFRY4X64_20 = 4, ORC_MTGP32 = 5 };
enum { ORC_SPACING_STREAM = 0, ORC_SPACING_SUBSTREAM = 1, ORC_SPACING_KEYED = 2, ORC_SPACING_LEAPFROG = 3 };
enum { ORC_U32 = 0, ORC_F32 = 1, ORC_F64 = 2 };

/* ---- MRG32k3a (P L250-282 §4.1; constants from [LEcuyer1999], P L255) ---- */
/* One step of the combined recurrence. s = (s10,s11,s12,s20,s21,s22), oldest
 * first (R1). Advances s in place and returns z in [1, m1] (R2). */
uint32_t orc_mrg_step(uint32_t s[6]);
/* The two 3x3 companion matrices A1 (mod m1) and A2 (mod m2), row-major. */
void orc_mrg_matrices(uint64_t A1[9], uint64_t A2[9]);
/* C = A*B mod m (3x3, row-major, entries < m). */
void orc_mat_mul(const uint64_t A[9], const uint64_t B[9], uint64_t m, uint64_t C[9]);
/* out = A^e mod m, e = e_hi*2^64 + e_lo, by square-and-multiply (P L112-117). */
void orc_mat_pow(const uint64_t A[9], uint64_t e_lo, uint64_t e_hi, uint64_t m, uint64_t out[9]);
/* s <- A^e s componentwise: the state after e steps (S L157-165). */
void orc_mrg_jump(uint32_t s[6], uint64_t e_lo, uint64_t e_hi);
/* State at position g*2^127 + u*2^76 + o of the sequence started at seed
 * (P L264-268; S L166-174): (A^(2^127))^g (A^(2^76))^u A^o seed. */
void orc_mrg_position(const uint32_t seed[6], uint64_t g, uint64_t u,
                      uint64_t o_lo, uint64_t o_hi, uint32_t out[6]);

/* ---- Philox4x32 (P L322-336 §4.3; constants from [Salmon.etal.2011]) ---- */
void orc_philox_block(const uint32_t ctr[4], const uint32_t key[2], int rounds,
                      uint32_t out[4]);

/* ---- Threefry4x64 (P L322-336 §4.3; [Salmon.etal.2011]) ---- */
void orc_threefry4x64_block(const uint64_t ctr[4], const uint64_t key[4], int rounds, uint64_t out[4]);

/* ---- TinyMT32 (P L287-317 §4.2; algorithm from [Saito2011], P L292) ---- */
/* State: status[4] plus the parameter set (mat1, mat2, tmat). */
typedef struct {
    uint32_t st[4];
    uint32_t mat1, mat2, tmat;
} orc_tinymt32;
void orc_tinymt32_init(orc_tinymt32* t, uint32_t mat1, uint32_t mat2, uint32_t tmat, uint32_t seed);
void orc_tinymt32_next_state(orc_tinymt32* t);
uint32_t orc_tinymt32_temper(const orc_tinymt32* t);
uint32_t orc_tinymt32_generate(orc_tinymt32* t); /* next_state then temper */
/* The transition is linear over GF(2) on the 128 status bits: jump e steps
 * by applying T^e, T built column by column from next_state of unit vectors
 * (e = e_hi*2^64 + e_lo, square-and-multiply; R15). */
void orc_tinymt32_jump(orc_tinymt32* t, uint64_t e_lo, uint64_t e_hi);

/* ---- MTGP32 (P L74-76 [§2.2], L133-136 [§2.3]; algorithm from
 * [Saito.Matsumoto2012], Mersenne exponent 11213: N = 11213/32 + 1 = 351
 * state words). Parameter set (one per state, the DC output; R18):
 * pos, sh1, sh2, mask, tbl[16], tmp_tbl[16]. ---- */
#define ORC_MTGP32_N 351
typedef struct {
    uint32_t pos, sh1, sh2, mask;
    uint32_t tbl[16], tmp_tbl[16];
} orc_mtgp32_params;
typedef struct {
    uint32_t x[ORC_MTGP32_N]; /* ring: x[(idx + k) % N] is the k-th oldest word */
    int idx;
    orc_mtgp32_params p;
} orc_mtgp32;
/* State from a 32-bit seed ([Saito.Matsumoto2012] init_state: hidden seed
 * from tbl[4], tbl[8]; byte fill; Knuth's 1812433253 recursion). */
void orc_mtgp32_init(orc_mtgp32* m, const orc_mtgp32_params* p, uint32_t seed);
/* x_{k+N} = rec(x_k, x_{k+1}, x_{k+pos}); output = temper(x_{k+N}, x_{k+pos-1}). */
uint32_t orc_mtgp32_generate(orc_mtgp32* m);

/* ---- conversions (R7) ---- */
float orc_to_f32(uint32_t w);
double orc_mrg_to_f64(uint32_t z);
double orc_philox_to_f64(uint32_t lo, uint32_t hi);

/* ---- streams: the paper's per-PE object with next() (P L387-399 §5.2) ---- */
typedef struct {
    int gen;
    uint32_t s[6];        /* MRG32k3a state */
    uint32_t key[2];      /* Philox key (R6) */
    orc_tinymt32 tm;      /* TinyMT32 state and parameters */
    orc_mtgp32 mt;        /* MTGP32 state and parameters */
    uint64_t g;           /* Philox stream index -> ctr[2..3] (R6) */
    uint64_t blk;         /* Philox next counter block -> ctr[0..1] (R6) */
    uint32_t buf[4];      /* Philox lanes not yet served (S L258-266) */
    int buf_pos;          /* next lane to serve; 4 = empty */
    uint64_t tkey[4];     /* Threefry key (R16) */
    uint32_t tbuf[8];     /* Threefry words not yet served; tpos = 8: empty */
    int tpos;
    uint64_t leap;        /* Leap Frog: players K (0: not a leap-frog stream) */
    uint64_t leapA1[9], leapA2[9]; /* MRG32k3a: A^(K-1), the K-1 skipped draws */
    uint64_t pos_lo, pos_hi;       /* counter-based: next base draw index */
    uint32_t leapT[128][4];        /* TinyMT32 Leap Frog: T^(K-1) columns (K > 65) */
} orc_stream;

/* Open handle-stream i of a (gen, seed, first, spacing) family at draw offset
 * (off_hi:off_lo). Returns 0 on success, -1 on invalid arguments.
 * TinyMT32 (R15): seed = {seed, group_size, n_params, mat1_0, mat2_0, tmat_0,
 * mat1_1, ...} (nseed = 3 + 3*n_params); family stream g = first + i lies in
 * group g / group_size, which uses parameter set g / group_size (one set per
 * group, P L309-313), and is slice g % group_size of that group's sequence,
 * i.e. starts 2^64 * (g % group_size) draws after init(params, seed).
 * MTGP32 (R18): seed = {seed_lo, seed_hi, n_params, then 36 words per
 * parameter set (pos, sh1, sh2, mask, tbl[16], tmp_tbl[16])}; family stream
 * g = first + i uses parameter set g (g < n_params; Parameterization, one
 * set per state, P L74-76) seeded with (uint32)(s ^ s >> 32) + g + 1,
 * s = seed_hi:seed_lo; the offset is reached by stepping (off < 2^64). */
int orc_stream_open(orc_stream* st, int gen, const uint32_t* seed, int nseed,
                    uint64_t first, uint64_t i, int spacing,
                    uint64_t off_lo, uint64_t off_hi);
uint32_t orc_stream_next(orc_stream* st);

/* Leap Frog (P L118-122 [§2.3]: "like a deck of cards dealt to card
 * players"; S L397, L424): one base sequence dealt round-robin to K players;
 * player p receives base draws p, p+K, p+2K, ... Its draw offset o counts its
 * own draws (base draw p + K*o is its next). Base sequence (R17): MRG32k3a
 * stream 0 of seed; Philox4x32-10 / Threefry4x64-20 counter stream 0 of key
 * seed. Each draw takes the next base draw, then skips K-1 base draws (MRG:
 * the jump A^(K-1), S L157-165; counter-based: the index advances by K).
 * TinyMT32 (R19): seed = {seed, mat1, mat2, tmat}, the base sequence is
 * init(params, seed); skips by stepping (K <= 65) or by the matrix T^(K-1).
 * Returns -1 if p >= K or the base sequence is exhausted at the start
 * position (Philox 2^66, Threefry 2^67, MRG 2^128 draws). */
int orc_stream_open_leapfrog(orc_stream* st, int gen, const uint32_t* seed, int nseed,
                             uint64_t players, uint64_t player, uint64_t off_lo, uint64_t off_hi);

/* Stream-major rows out[i*n + j] (R8) for streams i < n_streams; kind picks
 * u32 / f32 / f64 (Philox f64 consumes two draws per value, R7).
 * nthreads >= 1 splits streams into contiguous ranges (result independent
 * of nthreads). Returns 0 or -1. */
int orc_generate(int gen, const uint32_t* seed, int nseed, uint64_t first,
                 uint64_t n_streams, int spacing, uint64_t off_lo, uint64_t off_hi,
                 uint64_t n, int kind, void* out, int nthreads);

/* Monte Carlo pi dartboard (S L529-537; R9): sample k of stream i uses draws
 * 2k, 2k+1 from the offset; hit iff X^2+Y^2 < 2^48 with X = w>>8, Y = w'>>8.
 * counts[i] (if non-NULL) receives per-stream hits; returns the total. */
uint64_t orc_mc_count(int gen, const uint32_t* seed, int nseed, uint64_t first,
                      uint64_t n_streams, int spacing, uint64_t off_lo, uint64_t off_hi,
                      uint64_t samples, uint64_t* counts, int nthreads);
/* Same, but only for an explicit list of handle-stream indices. */
uint64_t orc_mc_count_list(int gen, const uint32_t* seed, int nseed, uint64_t first,
                           const uint64_t* idx, uint64_t n_idx, int spacing,
                           uint64_t off_lo, uint64_t off_hi, uint64_t samples,
                           uint64_t* counts, int nthreads);
/* Rows for an explicit list of handle-stream indices: out[r*n + j]. */
int orc_generate_list(int gen, const uint32_t* seed, int nseed, uint64_t first,
                      const uint64_t* idx, uint64_t n_idx, int spacing,
                      uint64_t off_lo, uint64_t off_hi, uint64_t n, int kind,
                      void* out, int nthreads);

/* Leap Frog rows / dartboard for players first + idx[r] (idx NULL: first + r,
 * r < n_rows) of K = players (see orc_stream_open_leapfrog). */
int orc_generate_leapfrog(int gen, const uint32_t* seed, int nseed, uint64_t players, uint64_t first,
                          const uint64_t* idx, uint64_t n_rows, uint64_t off_lo, uint64_t off_hi,
                          uint64_t n, int kind, void* out, int nthreads);
uint64_t orc_mc_count_leapfrog(int gen, const uint32_t* seed, int nseed, uint64_t players,
                               uint64_t first, const uint64_t* idx, uint64_t n_rows, uint64_t off_lo,
                               uint64_t off_hi, uint64_t samples, uint64_t* counts, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
