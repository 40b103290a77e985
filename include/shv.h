/*
 * shv.h — C ABI of the B200-native ShoveRand hot path (arXiv 1412.8266):
 * bulk generation of many independent, reproducible pseudorandom streams.
 *
 * Citations: "P Lnn" = PAPER.md line nn (section in brackets), "S Lnn" =
 * SPEC.md line nn, "Rk" = reading k in DESIGN.md §3 (the paper is silent or
 * ambiguous there). Library: paper_1412_8266_b200/libshv.so (sm_100a).
 *
 * Model of the problem (P L353-382 [§5.1], L480-499 [Listing 1]): the caller
 * states only how much parallelism it needs (n_streams); the library owns the
 * distribution of the random sequence over those streams (Sequence Splitting,
 * P L109-112 [§2.3]) and keeps the user's buffers and kernels free of generator
 * plumbing. Handle stream i < n_streams is
 *   MRG32k3a, SHV_SPACING_STREAM    : stream first+i, 2^127 draws apart  (P L264-268 [§4.1])
 *   MRG32k3a, SHV_SPACING_SUBSTREAM : substream first+i of stream 0, 2^76 apart (ibid.)
 *   Philox4x32-10, SHV_SPACING_STREAM: counter-stream g = first+i, counter
 *                                     (blk_lo, blk_hi, g_lo, g_hi), key = seed (P L322-336 [§4.3]; R6)
 *   Philox4x32-10, SHV_SPACING_KEYED : key = (first+i, tag), counter (blk_lo, blk_hi, 0, 0)
 *   Threefry4x64-20 (STREAM)        : ctr = (blk, first+i, 0, 0), key from the seed words (R16)
 *   TinyMT32 (shv_streams_create_tinymt32): parameter set per group, 2^64-draw slices (R15)
 *   SHV_SPACING_LEAPFROG (shv_streams_create_leapfrog): player first+i of K
 *                                     receives base draws p, p+K, ... (P L118-122 [§2.3]; R17)
 * Every stream of a handle sits at the same draw offset o (u128), which each
 * generate / mc_pi call advances by the draws it consumed (S L58; R8).
 *
 * Conventions for every call:
 *  - extern "C", no exceptions escape, never aborts, does not change the
 *    calling thread's current CUDA device (it is saved and restored).
 *  - Device pointers are plain CUDA device addresses (e.g. torch
 *    tensor.data_ptr()) on the handle's device; the caller owns them and keeps
 *    them alive until the work queued on cuda_stream has completed.
 *  - cuda_stream is a cudaStream_t (NULL = legacy default stream). Kernel work
 *    is stream-ordered and asynchronous; host-side validation is synchronous.
 *  - A call that returns an error has no side effects (no launch, no offset
 *    change), except SHV_ERR_CUDA, which reports an error the CUDA runtime
 *    raised while enqueueing. shv_last_error_message() gives detail
 *    (thread-local).
 *  - Handles are opaque non-zero ids in a mutex-protected registry; a handle
 *    must not be used concurrently from two host threads (S L96).
 */
#ifndef SHV_H
#define SHV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SHV_OK = 0,
    SHV_ERR_INVALID_ARGUMENT = 1,     /* bad enum, NULL out-pointer, size overflow, stream exhausted */
    SHV_ERR_INVALID_SEED = 2,         /* S L50, L117-118: residue >= m, or an all-zero MRG triple */
    SHV_ERR_INSUFFICIENT_STREAMS = 3, /* S L50, L199-200: first+n beyond 2^64 streams / 2^51 substreams */
    SHV_ERR_UNSUPPORTED = 4,          /* combination the generator does not define (Philox substreams) */
    SHV_ERR_LIFECYCLE = 5,            /* S L67-72: unknown, destroyed or double-destroyed handle */
    SHV_ERR_MISALIGNED = 6,           /* output pointer not aligned to its element size */
    SHV_ERR_EMPTY_EXPERIMENT = 7,     /* S L535: Monte Carlo with zero samples */
    SHV_ERR_MISSING_PARAMETERS = 8,   /* reserved for parameter-file generators (TinyMT, MTGP) */
    SHV_ERR_CUDA = 9                  /* CUDA runtime error while enqueueing */
} shv_status;

typedef enum {
    SHV_GEN_MRG32K3A = 1,       /* [LEcuyer1999], P L82-86, L250-282 [§4.1] */
    SHV_GEN_PHILOX4X32_10 = 2,  /* [Salmon.etal.2011], P L88-90, L322-336 [§4.3]; variant per S L275 */
    SHV_GEN_TINYMT32 = 3,       /* [Saito2011], P L287-317 [§4.2]; shv_streams_create_tinymt32 */
    SHV_GEN_MTGP32 = 5,         /* [Saito.Matsumoto2012], P L74-76 [§2.2], L133-136 [§2.3]:
                                   MTGP32-11213, one Dynamic Creator parameter set per stream;
                                   shv_streams_create_mtgp32 (R18) */
    SHV_GEN_THREEFRY4X64_20 = 4 /* [Salmon.etal.2011], P L322-336 [§4.3]; variant per S L275;
                                   key = (s0|s1<<32, s2|s3<<32, 0, 0) from 1..4 seed words,
                                   counter-stream g: ctr = (blk, g, 0, 0); draws are the (lo, hi)
                                   32-bit words of the four 64-bit lanes (R16); STREAM spacing only */
} shv_gen;

typedef enum {
    SHV_SPACING_STREAM = 0,     /* MRG: 2^127 draws apart; Philox: counter-stream index */
    SHV_SPACING_SUBSTREAM = 1,  /* MRG: 2^76 draws apart; Philox: SHV_ERR_UNSUPPORTED */
    SHV_SPACING_KEYED = 2,      /* Philox only: Parameterization, one key per stream
                                   (P L331-334 "a single key that can be set at runtime
                                   according to each thread's unique identifier"; S L249-257):
                                   key = (first+i, tag), counter = (blk_lo, blk_hi, 0, 0);
                                   seed = 1 word, the experiment tag; first+n <= 2^32
                                   (else SHV_ERR_INSUFFICIENT_STREAMS, S L253 KeySpaceExhausted).
                                   MRG: SHV_ERR_UNSUPPORTED */
    SHV_SPACING_LEAPFROG = 3    /* Leap Frog partition; handles from shv_streams_create_leapfrog */
} shv_spacing;

typedef enum {
    SHV_JUMP_DRAWS = 0,         /* o += n                            */
    SHV_JUMP_SUBSTREAMS = 1,    /* o += n * 2^76  (MRG only)         */
    SHV_JUMP_STREAMS = 2        /* o += n * 2^127 (MRG only)         */
} shv_jump_kind;

typedef uint64_t shv_streams; /* registry id; 0 is never valid */

/* Checkpoint record (S L98-99, L193-194): a stream family is a pure function
 * of these fields, so create_ex + shv_jump(offset) resumes bit-exactly. */
typedef struct {
    uint32_t gen, spacing;
    uint32_t seed[6];     /* MRG: s10 s11 s12 s20 s21 s22; Philox: key0 key1 0 0 0 0 */
    uint64_t first_stream, n_streams;
    uint64_t offset_lo, offset_hi;
    uint64_t players;     /* SHV_SPACING_LEAPFROG: K; otherwise 0 */
} shv_position;

/* Bytes of per-stream state a handle needs: MRG32k3a 24*n_streams (six u32
 * per stream, SoA: word k of stream i at [k*n_streams + i]; P L257-258
 * "only stores 6 integers"); Philox 0 (counter-based, no state); TinyMT32 16;
 * MTGP32 1408 (352 words per stream). */
size_t shv_state_bytes(int gen, uint64_t n_streams);

/* Short form (north star): first_stream 0, SHV_SPACING_STREAM, current
 * device, legacy default stream, library-allocated state (cudaMalloc, freed
 * by shv_streams_destroy). Host-synchronous. */
shv_status shv_streams_create(shv_streams* out, int gen, const uint32_t* seed,
                              size_t seed_words, uint64_t n_streams);

/* Full form (P L358-382 [§5.1] init(block_num)).
 *  seed/seed_words: MRG32k3a 1 word v (all six residues = v) or 6 words
 *    s10 s11 s12 s20 s21 s22 (S L114-119); Philox 1 or 2 words key0[, key1]
 *    (key1 = 0 if omitted). Anything else: SHV_ERR_INVALID_ARGUMENT.
 *  first_stream, n_streams: handle stream i is family stream first_stream+i.
 *    n_streams >= 1.
 *  spacing: see shv_spacing.
 *  d_state: MRG only — device buffer of state_bytes >= shv_state_bytes(),
 *    4-byte aligned, owned by the caller until destroy; NULL lets the library
 *    allocate it. Ignored for Philox.
 *  device: CUDA device ordinal the handle lives on (-1 = current device).
 *  cuda_stream: the per-stream seeding kernel (start state = product of
 *    host-built jump matrices applied to the seed, P L264-268) is enqueued
 *    here; the first create on a device also uploads the jump tables
 *    synchronously. */
shv_status shv_streams_create_ex(shv_streams* out, int gen, const uint32_t* seed,
                                 size_t seed_words, uint64_t first_stream, uint64_t n_streams,
                                 int spacing, void* d_state, size_t state_bytes, int device,
                                 void* cuda_stream);

/* Advance every stream of the handle by n draws, substreams or streams
 * (jump-ahead, P L112-117 [§2.3]; S L157-174): kind = SHV_JUMP_DRAWS /
 * SUBSTREAMS / STREAMS, see shv_jump_kind. Stream-ordered on cuda_stream like
 * generate: for MRG32k3a, Philox, Threefry and every Leap Frog handle the jump
 * is host-side only (the handle's offset; the next launch starts there); for
 * the stateful TinyMT32 and MTGP32 handles the state buffer is advanced by a
 * kernel enqueued on cuda_stream, ordered with the caller's generate / mc_pi
 * calls on that stream (TinyMT32: any n, by the jump polynomial x^n mod the
 * minimal polynomial of each group's transition; MTGP32: sequential steps).
 * Errors: UNSUPPORTED for Philox sub/streams; INVALID_ARGUMENT if the offset
 * would leave the stream (Philox 2^66 draws; MRG offset beyond 2^128). */
shv_status shv_jump(shv_streams h, int kind, uint64_t n, void* cuda_stream);

/* TinyMT32 handles (NEXT-3; P L287-317 [§4.2]; R15) — the paper's hybrid:
 * one Dynamic Creator parameter set per group of group_size streams ("the
 * same independent parameterized status is shared among all the threads of a
 * CUDA block", P L309-313), and inside a group, stream s is slice s of the
 * group's sequence: 2^64 draws per slice after the authors' init(params, seed)
 * ("the original stream is sliced in equal chunks", P L313-317).
 *  params: n_params records (mat1, mat2, tmat), host memory, DC output supplied
 *    by the caller (P L304-306); family stream g = first+i uses record g/group_size.
 *  group_size: power of two <= 2^16 (slice starts via GF(2) jump matrices
 *    built on the device at create).
 *  d_state: 16*n_streams bytes (SoA, four words per stream) or NULL.
 * The handle is stateful: generate/mc_pi advance the state buffer in place;
 * shv_jump(DRAWS, n) advances the states on the jump's cuda_stream.
 * TinyMT f64 values use two draws, like Philox (R7). Errors: params NULL or
 * n_params 0 -> SHV_ERR_MISSING_PARAMETERS; groups beyond n_params ->
 * SHV_ERR_INSUFFICIENT_STREAMS. Host-synchronous (waits for seeding). */
shv_status shv_streams_create_tinymt32(shv_streams* out, const uint32_t* params, size_t n_params,
                                       uint32_t seed, uint32_t group_size, uint64_t first_stream,
                                       uint64_t n_streams, void* d_state, size_t state_bytes,
                                       int device, void* cuda_stream);

/* Leap Frog handles (NEXT-4; P L118-122 [§2.3]: "Assigning random sequences
 * ... like a deck of cards dealt to card players"; S L397-424; R17). One base
 * sequence is dealt round-robin to `players` (K >= 1) players: handle stream i
 * is player p = first_player + i and its draw t is base draw p + K*t (t counted
 * from the handle offset o, which counts the player's own draws). Base
 * sequence: MRG32k3a stream 0 of the seed (seed words as create_ex);
 * Philox4x32-10 / Threefry4x64-20 counter stream 0 of the key (ctr[2..3] = 0
 * resp. ctr[1] = 0); TinyMT32 (R19): seed_words = 4, {seed, mat1, mat2, tmat},
 * the authors' init(params, seed) sequence (player states reached with GF(2)
 * jump tables built on the device at create; each draw skips K - 1 base draws
 * by stepping for K <= 65, else by the matrix T^(K-1); fewer than 4 words:
 * SHV_ERR_MISSING_PARAMETERS); MTGP32: SHV_ERR_UNSUPPORTED. first_player + n_players
 * must be <= players (else SHV_ERR_INSUFFICIENT_STREAMS). generate_* and
 * mc_pi* work as for any handle (f64 / MC consume the player's own draws,
 * R7, R9); shv_jump takes SHV_JUMP_DRAWS only (player draws); a call whose
 * last base draw would leave the base stream (Philox 2^66, Threefry 2^67,
 * MRG 2^128 draws) fails with SHV_ERR_INVALID_ARGUMENT. The device view
 * (shv_get_device_view) is SHV_ERR_UNSUPPORTED for these handles.
 *  d_state: MRG32k3a only, shv_state_bytes(MRG, n_players) bytes or NULL: the
 *    base state A^p * seed of each player (SoA, P L257-258), seeded on
 *    cuda_stream as in create_ex. Kernels step a player with the order-3
 *    recurrence that A^K's characteristic polynomial gives each component
 *    (DESIGN.md §4.6): 6 modular products per draw for any K. */
shv_status shv_streams_create_leapfrog(shv_streams* out, int gen, const uint32_t* seed,
                                       size_t seed_words, uint64_t players, uint64_t first_player,
                                       uint64_t n_players, void* d_state, size_t state_bytes,
                                       int device, void* cuda_stream);

/* Bulk fill (P L485-490 [Listing 1] with n_per_stream draws per stream):
 * d_out[i*n + j] = value of draw o+j of stream i (f64 Philox: draws o+2j,
 * o+2j+1), for i < n_streams, j < n; then o += n (Philox f64: 2n). Row-major,
 * stream-major (R8). Values (R7):
 *   u32: the generator word (MRG: z in [1, m1]; Philox: lane x,y,z,w order);
 *   f32: (w >> 8) * 2^-24 in [0,1), exact;
 *   f64: MRG fl64(z * 0x1.000000d00000bp-32) in (0,1); Philox
 *        ((w_{2j+1} << 32 | w_{2j}) >> 11) * 2^-53 in [0,1), exact.
 * d_out must be aligned to the element size (else SHV_ERR_MISALIGNED); a
 * 32-byte aligned pointer with 32-byte rows takes the vectorised path, any
 * other shape a scalar path with identical values. n = 0 is a no-op. */
shv_status shv_generate_u32(shv_streams h, uint32_t* d_out, uint64_t n_per_stream, void* cuda_stream);
shv_status shv_generate_f32(shv_streams h, float* d_out, uint64_t n_per_stream, void* cuda_stream);
shv_status shv_generate_f64(shv_streams h, double* d_out, uint64_t n_per_stream, void* cuda_stream);

/* MTGP32-11213 handle (NEXT-4c; Parameterization, P L74-76 [§2.2]: "MTGP
 * ... comes with companion software for parallelization (MTGPDC)";
 * P L133-136; R18). params: n_params records of 36 u32 words, the Dynamic
 * Creator output for Mersenne exponent 11213 — pos, sh1, sh2, mask,
 * tbl[16], tmp_tbl[16] (e.g. the 200 sets of the CUDA toolkit's
 * curand_mtgp32dc_p_11213.h); host memory, copied. Family stream g =
 * first_stream + i (i < n_streams) uses parameter set g, so
 * first_stream + n_streams <= n_params (else SHV_ERR_INSUFFICIENT_STREAMS),
 * and starts from the authors' init_state(params[g], (uint32)(s ^ s >> 32)
 * + g + 1), s = seed (the convention of cuRAND's
 * curandMakeMTGP32KernelState). The handle is stateful: 1408 bytes per stream
 * (shv_state_bytes; d_state as in shv_streams_create_ex), rewritten by every
 * generate / mc_pi call and by shv_jump (SHV_JUMP_DRAWS only; sequential
 * advance enqueued on the create stream). f32/f64/Monte Carlo conversions
 * as for Philox (R7, R9: f64 and each sample take two draws). No device view
 * and no Leap Frog layout (SHV_ERR_UNSUPPORTED): MTGP32 is generated by the
 * threads of a block together. Errors: NULL params ->
 * SHV_ERR_MISSING_PARAMETERS; a record with pos outside [3, 349] or a shift
 * above 31 -> SHV_ERR_INVALID_ARGUMENT. */
shv_status shv_streams_create_mtgp32(shv_streams* out, const uint32_t* params, size_t n_params,
                                     uint64_t seed, uint64_t first_stream, uint64_t n_streams,
                                     void* d_state, size_t state_bytes, int device, void* cuda_stream);

/* Same values as shv_generate_u32, written to a HOST buffer h_out (pinned
 * memory recommended). The library generates into device staging slices and
 * copies them back on an internal copy stream overlapped with generation;
 * completion is ordered on cuda_stream (synchronize it before reading). */
shv_status shv_generate_u32_host(shv_streams h, uint32_t* h_out, uint64_t n_per_stream, void* cuda_stream);

/* Fused Monte Carlo pi dartboard (P L18-21 [§1], S L529-537; R9): sample k of
 * stream i uses draws o+2k, o+2k+1; X = w>>8, Y = w'>>8; hit iff
 * X^2 + Y^2 < 2^48. Numbers never touch memory. *d_hits (device u64, zeroed
 * by the caller) += total hits over the handle's streams; o += 2*samples.
 * pi_hat = 4 * hits / (n_streams * samples). samples = 0:
 * SHV_ERR_EMPTY_EXPERIMENT. d_stream_counts (optional, _ex only): device u64
 * per stream, += that stream's hits (used by parity tests). */
shv_status shv_mc_pi(shv_streams h, uint64_t samples_per_stream, uint64_t* d_hits, void* cuda_stream);
shv_status shv_mc_pi_ex(shv_streams h, uint64_t samples_per_stream, uint64_t* d_hits,
                        uint64_t* d_stream_counts, void* cuda_stream);

shv_status shv_get_position(shv_streams h, shv_position* out);

/* Device-side view of a handle for user kernels (the paper's device API,
 * P L387-399 [§5.2], Listing 1 P L485-490): pass it by value to a kernel and
 * construct shv::Rng<GEN>(view, i) from include/shv_rng.cuh in each thread;
 * rng.next_u32()/next_f32()/next_f64() then produce exactly the values
 * shv_generate_* would write for stream i at the handle's current offset
 * (R7, R8). The view is a snapshot: after a kernel consumed up to K draws per
 * stream, advance the handle with shv_jump(h, SHV_JUMP_DRAWS, K). The state
 * pointer stays valid until shv_streams_destroy. */
typedef struct {
    uint32_t gen, spacing;
    uint32_t key0, key1;          /* Philox key words (keyed: key1 = tag) */
    uint64_t first_stream, n_streams;
    uint64_t offset_lo, offset_hi;
    const uint32_t* state;        /* MRG: SoA start states (offset 0); TinyMT: current states; NULL for Philox */
    uint32_t jump[18];            /* MRG: A1^o (mod m1), A2^o (mod m2), row-major */
    const uint32_t* params;       /* TinyMT: (mat1, mat2, tmat) per group from group0 */
    uint64_t group0;              /* TinyMT: first group of the handle */
    uint32_t group_size;          /* TinyMT */
    uint32_t key2, key3;          /* Threefry key words 2, 3 */
} shv_device_view;

shv_status shv_get_device_view(shv_streams h, shv_device_view* out);

/* Release (P L498 [Listing 1] release()). Frees library-allocated state with
 * cudaFree (which synchronizes the device); the id becomes invalid, a second
 * destroy returns SHV_ERR_LIFECYCLE (S L67-72). */
shv_status shv_streams_destroy(shv_streams h);

const char* shv_status_string(shv_status s);
const char* shv_last_error_message(void);

/* ---- disjointness audit (S L407-415 [partition: verify_disjoint], L425-426) ----
 * Audits rows that were generated for n_pe processing elements (e.g. the
 * d_out of shv_generate_u32: row i = the draws of stream i; P L109-122 [§2.3]
 * "non-overlapping contiguous blocks"): every window of 4 consecutive u32
 * draws of every row is hashed into a table in d_workspace, and a window value
 * held by two DIFFERENT rows is a collision (single-word coincidences are
 * expected by birthday statistics and prove nothing, S L426).
 *   d_rows      device u32[n_pe * horizon], row-major (row i at i*horizon);
 *   horizon     draws per PE; rows shorter than 4 have no windows;
 *   d_workspace device scratch of workspace_bytes, 8-byte aligned, at least
 *               shv_verify_disjoint_workspace_bytes(n_pe, horizon) bytes
 *               (48 bytes per window + 40 per hash bucket + 48: the records,
 *               the bucket tables at load <= 1/2 and the candidate list);
 *   d_report    device shv_disjoint_report, written stream-ordered.
 * The report is a function of the rows alone (deterministic merge, S L429):
 * if not disjoint, (pe_a, pos_a, pe_b, pos_b) is the lexicographically
 * smallest over all pairs of equal windows with pe_a < pe_b; otherwise those
 * four fields are ~0. Runs on the CURRENT CUDA device (all three pointers must
 * be on it). Errors: NULL pointers or n_pe * horizon >= 2^40 ->
 * SHV_ERR_INVALID_ARGUMENT; workspace too small -> SHV_ERR_INVALID_ARGUMENT;
 * misaligned workspace or report -> SHV_ERR_MISALIGNED. */
typedef struct {
    uint64_t disjoint;    /* 1: no window value is held by two different PEs */
    uint64_t windows;     /* n_pe * (horizon - 3), 0 if horizon < 4 */
    uint64_t colliding;   /* distinct window values held by >= 2 different PEs */
    uint64_t pe_a, pos_a; /* first collision (see above) */
    uint64_t pe_b, pos_b;
} shv_disjoint_report;

size_t shv_verify_disjoint_workspace_bytes(uint64_t n_pe, uint64_t horizon);
shv_status shv_verify_disjoint(const uint32_t* d_rows, uint64_t n_pe, uint64_t horizon,
                               void* d_workspace, size_t workspace_bytes,
                               shv_disjoint_report* d_report, void* cuda_stream);

/* ---- launch configuration (results never depend on it; R10) ---- */
/* Override the persistent-grid shape and work split of one handle:
 * blocks_per_sm (0 = occupancy maximum), threads_per_block (0 = 256,
 * else a multiple of 32 in [32, 256]), segment (0 = automatic; else the
 * number of draws-per-value units one work item covers, a multiple of 8). */
shv_status shv_set_launch_config(shv_streams h, uint32_t blocks_per_sm,
                                 uint32_t threads_per_block, uint64_t segment);

/* ---- host-only utilities (no GPU needed) ---- */
/* Rank r of world w owns handle streams [*first, *first + *count) of a
 * family of total_streams (contiguous split). */
shv_status shv_partition(uint64_t total_streams, int rank, int world,
                         uint64_t* first, uint64_t* count);
/* The host-built jump matrices the kernels use: out[0..8] = A1^e mod m1,
 * out[9..17] = A2^e mod m2 (row-major), e = e_hi*2^64 + e_lo (S L148-156). */
shv_status shv_jump_matrix(uint64_t e_lo, uint64_t e_hi, uint32_t out[18]);
/* Library version string and the sm_ architecture it was built for. */
const char* shv_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SHV_H */
