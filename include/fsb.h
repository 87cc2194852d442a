/*
 * fsb.h -- C ABI of libfsb200.so, the B200-native Founsure 1.0 encode path
 * (arXiv 1702.07409).  Plain C types only: host pointers, device pointers, sizes.
 *
 * What the library computes (§2.2, Fig. 1, steps (1) and (2)):
 *
 *   precode ("Check #1"):  C_i = XOR_{m in P(i)} D_m            for i < p
 *   LT / LDGM stage:       Y_j = XOR_{m in N(j)} I_m            for j < n,
 *                          I = [D_0 .. D_{k-1}, C_0 .. C_{p-1}]  (K = k+p symbols)
 *
 * bytewise over t-byte symbols, for every stripe ("partition") with the
 * same graph.  The graph is drawn from a seeded PRNG: every check has d_p
 * distinct data neighbours; every coded symbol has a degree drawn from the Robust Soliton
 * distribution or a finite max-degree Omega(x), and that
 * many distinct neighbours among the K intermediate symbols.  Conventions for everything
 * the paper leaves open (PRNG, sampling, CDF arithmetic, stream order) are DESIGN.md §3
 * readings R2-R15.
 *
 * Notation: k = data symbols (paper b), p = precode checks (paper k-b),
 * n = coded symbols, t = bytes per symbol, S = stripes.
 *
 * Memory layout of every symbol block: symbol-major, t contiguous bytes per symbol
 * (reading R13).  Data of stripe s starts at d_data + s*data_stride, etc.
 *
 * Ownership: the library owns fs_graph (host CSR, device CSR, device work schedules,
 * allocated on the device current at creation) and the decode/repair plans (and, for
 * FS_DECODE_ELIMINATE plans, their device workspace, allocated on first use).  The caller
 * owns every data / check / coded buffer.  The library never allocates caller-visible memory
 * and never synchronises the caller's stream (except when a plan's workspace grows);
 * kernels are enqueued on the stream given.  Encode / decode / repair calls must be made
 * with the object's device current (else FS_EINVAL).
 *
 * Errors: every call returns fs_status (0 = OK).  Validation failures return FS_EINVAL /
 * FS_EDIST without side effects; launch failures return FS_ECUDA.  Asynchronous kernel
 * faults surface at the caller's next synchronisation.  fs_last_error() returns a
 * thread-local message describing the last failure on the calling thread.
 *
 * Thread safety: a graph is immutable after creation (except fs_graph_set_variant, which
 * must not race with encodes); concurrent fs_encode* calls on different streams are fine.
 * Plans cache a CUDA graph of their level launches and their workspace under an internal
 * mutex (host calls on one plan are serialised); a plan with a workspace (FS_DECODE_ELIMINATE)
 * must not run on two streams at once -- order such calls (one stream, or events).
 * Output is deterministic and independent of stream, launch configuration, kernel
 * variant and GPU count (XOR is exact, associative and commutative).
 */
#ifndef FSB_H_
#define FSB_H_

#include <stdint.h>

#if defined(__GNUC__)
#define FSB_API __attribute__((visibility("default")))
#else
#define FSB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FS_OK = 0,
  FS_EINVAL = -1,       /* invalid argument (sizes, alignment, strides, pointers)          */
  FS_EDIST = -2,        /* invalid degree distribution                                    */
  FS_ENOMEM = -3,       /* host or device allocation failed                                */
  FS_ECUDA = -4,        /* CUDA runtime / launch error (message in fs_last_error())        */
  FS_EUNSUPPORTED = -5  /* operation not available for this graph (e.g. host-only graph)   */
} fs_status;

typedef enum { FS_DIST_RSD = 1, FS_DIST_FINITE = 2 } fs_dist_kind;

/* Precode kinds (PAPER.md:91 step (1), "Check #1").
 * FS_PRECODE_RANDOM: p checks, each the XOR of d_p distinct data symbols drawn from the graph
 *   stream (BASELINE.json configs; readings R5, R11).
 * FS_PRECODE_ARRAY: the paper's binary array LDPC precode, Alg 2 (SURVEY.md
 *   NEXT-2): for the paper's (b, k) = (k, k+p), P = largest prime factor of k+p, k' = (k+p)/P,
 *   j' = k' - k/P; p = j'P checks of k'-j' members each (data symbols or EARLIER checks), no
 *   stream draws; d_p is ignored (set to k'-j').  Realizable iff P divides k, j' >= 1,
 *   k' > j' and k' <= P (Alg 3's conditions); otherwise FS_EINVAL.                           */
typedef enum { FS_PRECODE_RANDOM = 0, FS_PRECODE_ARRAY = 1 } fs_precode_kind;

/* Code parameters: the paper's problem statement. */
typedef struct {
  uint32_t k;             /* data symbols (paper b); >= 1                                     */
  uint32_t p;             /* precode checks (paper k-b); 0 = no precode                       */
  uint32_t d_p;           /* data neighbours per check; 1 <= d_p <= k when p > 0             */
  uint32_t n;             /* coded symbols; >= 1                                              */
  uint64_t t;             /* bytes per symbol; multiple of 16, below 2^31                     */
  int32_t dist;           /* fs_dist_kind                                                     */
  double rsd_c;           /* RSD: c > 0                                                       */
  double rsd_delta;       /* RSD: 0 < delta < 1                                               */
  const uint32_t *fin_deg;   /* FINITE: support degrees, strictly increasing, >= 1           */
  const double *fin_prob;    /* FINITE: weights >= 0, sum within 1e-5 of 1 (normalised)      */
  uint32_t fin_len;          /* FINITE: number of support points                             */
  uint64_t seed;          /* splitmix64 graph seed (reading R2/R3)                            */
  int32_t precode;        /* fs_precode_kind (0 = FS_PRECODE_RANDOM)                          */
  uint32_t files;         /* s output files: 0 or 1 = one stream for all rows;
                             s > 1 (s | n): rows [i n/s, (i+1) n/s) of file i drawn from a stream
                             seeded seed + i (file 0 continues the base stream; reading R17)    */
} fs_params;

typedef struct fs_graph fs_graph;  /* opaque */

/* Graph-creation flags. */
#define FS_GRAPH_HOST_ONLY 1u   /* build host CSR only: no device memory, no CUDA calls.
                                   fs_encode* then return FS_EUNSUPPORTED.               */

/* Kernel variants (fs_graph_set_variant).  All produce identical bytes. */
#define FS_VARIANT_AUTO 0       /* per call: SMEM when the graph is eligible and the call
                                   covers all rows on 64-B slice boundaries, else GLOBAL */
#define FS_VARIANT_SMEM 1       /* persistent TMA-staged shared-memory tile kernel        */
#define FS_VARIANT_GLOBAL 2     /* L2-resident band sweep (precode kernel + LT kernel)    */

/* Seeded graph generation (step a1): precode rows first, then LT rows (reading R5), each
 * neighbour list sorted ascending (R14).  Without FS_GRAPH_HOST_ONLY the CSR and the work
 * schedules are uploaded to the current device (synchronously, before return).
 * FS_EINVAL: k == 0, n == 0, t == 0, t % 16 != 0 or t >= 2^31, p > 0 with d_p == 0 or d_p > k,
 *            K = k+p >= 2^31, files > 1 not dividing n.
 * FS_EDIST:  empty support, degree 0, degrees not strictly increasing, negative weight,
 *            |sum - 1| > 1e-5, RSD c <= 0, delta outside (0,1), R/delta <= 1, K/R < 1.   */
FSB_API fs_status fs_graph_create(const fs_params *prm, uint32_t flags, fs_graph **out);

/* Build a graph from CSR arrays (e.g. received by NCCL broadcast from rank 0).
 * pre_row_ptr[p+1], pre_col[p*d_p] (indices in [0,k), or k+i' for an earlier check i' < i),
 * lt_row_ptr[n+1], lt_col[nnz] (indices in [0,K)); rows need not be sorted but must hold
 * distinct indices, and precode levels must not decrease with the row index.
 * The arrays are copied.  FS_EINVAL on any structural violation.                         */
FSB_API fs_status fs_graph_from_csr(const fs_params *prm, const int32_t *pre_row_ptr,
                            const int32_t *pre_col, const int32_t *lt_row_ptr,
                            const int32_t *lt_col, uint32_t flags, fs_graph **out);

/* Host views of the graph's CSR (owned by g, valid until fs_free(g)).  Any out pointer may
 * be NULL.  pre_* are NULL-or-empty when p == 0.                                            */
FSB_API fs_status fs_graph_csr(const fs_graph *g, const int32_t **pre_row_ptr, const int32_t **pre_col,
                       const int32_t **lt_row_ptr, const int32_t **lt_col, uint64_t *lt_nnz);

/* Summary numbers of a graph (for rooflines and reports). */
typedef struct {
  uint32_t k, p, d_p, n;
  uint64_t t;
  uint64_t lt_nnz;           /* edges of the LT graph                                         */
  uint64_t pre_nnz;          /* edges of the precode graph (p*d_p)                            */
  uint32_t max_degree;       /* largest LT row degree                                         */
  int32_t variant;           /* FS_VARIANT_* currently set                                    */
  int32_t smem_eligible;     /* 1 when the SMEM variant can run this graph                    */
  uint32_t smem_bytes;       /* dynamic shared memory of the SMEM kernel                      */
  uint32_t sched_bytes;      /* size of the SMEM kernel's work schedule                       */
  uint32_t sched_steps_max;  /* SMEM schedule: gather slots of the most loaded warp per tile  */
  uint32_t sched_steps_avg;  /* SMEM schedule: mean gather slots per warp per tile (rounded)  */
  int32_t device;            /* CUDA device of the device copy, -1 for host-only graphs       */
  uint32_t lt_windows;       /* fixed-size LT edge windows of the GLOBAL window kernel (0: none,
                                i.e. a row of more than 93 edges; fs_graph_windows)              */
} fs_graph_info;

FSB_API fs_status fs_graph_get_info(const fs_graph *g, fs_graph_info *info);

/* Force a kernel variant (FS_VARIANT_*).  FS_EUNSUPPORTED if SMEM is requested for a graph
 * that is not eligible (t % 64 != 0, n > 65534, K+2 > 2047 tile rows, or two 64-B tiles plus
 * the schedule do not fit shared memory).                                                                */
FSB_API fs_status fs_graph_set_variant(fs_graph *g, int32_t variant);

/* One stripe, coded rows [row_begin, row_end) (row partition across GPUs).
 * d_data:   k*t bytes on the graph's device, 16-B aligned.
 * d_checks: p*t bytes (all p checks are always computed and written); NULL iff p == 0.
 * d_coded:  (row_end-row_begin)*t bytes; row j is written at d_coded + (j-row_begin)*t.
 * stream:   a cudaStream_t (NULL = legacy default stream).
 * Launches: GLOBAL = 1 precode kernel (if p > 0) + 1 LT kernel; SMEM = 1 fused kernel.   */
FSB_API fs_status fs_encode(const fs_graph *g, const uint8_t *d_data, uint8_t *d_checks,
                    uint8_t *d_coded, uint32_t row_begin, uint32_t row_end, void *stream);

/* fs_encode restricted to bytes [col_begin, col_end) of every symbol (byte-
 * range partition of a single large stripe across GPUs -- each rank reads and writes only its
 * columns, so unlike the row partition nothing is replicated).  Buffers are full-size as in
 * fs_encode (symbol stride t); bytes outside the range are neither read nor written.  The p checks
 * are computed for the range.  col_begin <= col_end <= t, multiples of 16, else FS_EINVAL.
 * Takes the SMEM variant only for full row ranges on 64-B slice boundaries.                  */
FSB_API fs_status fs_encode_range(const fs_graph *g, const uint8_t *d_data, uint8_t *d_checks,
                                  uint8_t *d_coded, uint32_t row_begin, uint32_t row_end,
                                  uint64_t col_begin, uint64_t col_end, void *stream);

/* num_stripes stripes with the same graph.  Strides are in bytes and must be
 * multiples of 16 and >= k*t, p*t, n*t respectively.  0 stripes is a no-op.               */
FSB_API fs_status fs_encode_stripes(const fs_graph *g, uint32_t num_stripes,
                            const uint8_t *d_data, uint64_t data_stride,
                            uint8_t *d_checks, uint64_t checks_stride,
                            uint8_t *d_coded, uint64_t coded_stride, void *stream);

/* fs_encode_stripes with the buffers in HOST memory: the library stages them through device
 * memory it owns (allocated on first use, kept with g, freed by fs_free) and overlaps the copies
 * in both directions with the kernels, in `chunks` pieces (0 = 32) issued alternately on two
 * library streams: whole stripes when num_stripes > 1, byte columns (>= 2 KB, the
 * fs_encode_range partition) for a single stripe.  Strides as for fs_encode_stripes (host
 * layout [stripe][symbol][t]; for one stripe the symbols are contiguous, stride t).  Host
 * buffers should be page-locked (cudaHostAlloc / cudaHostRegister) for the copies to overlap;
 * pageable memory works but serialises.  Enqueued after the work already on `stream`; `stream`
 * continues only after all of it, so the host buffers must stay valid and untouched until the
 * caller synchronises `stream`.  Calls on one graph are serialised with each other, so each call
 * fills and drains its own pipeline (measured, config 4: 39.1 GB/s end to end at 32 chunks vs
 * 39.8 for chunks of consecutive calls interleaved on the caller's side).
 * FS_EINVAL on NULL / misaligned-stride arguments or a host-only graph (FS_EUNSUPPORTED).      */
FSB_API fs_status fs_encode_host(const fs_graph *g, uint32_t num_stripes,
                                 const uint8_t *h_data, uint64_t data_stride,
                                 uint8_t *h_checks, uint64_t checks_stride,
                                 uint8_t *h_coded, uint64_t coded_stride, uint32_t chunks, void *stream);

/* Diagnostic view of the SMEM kernel's host-built LT schedule (owned by g):
 * words[nwords] = two chunk streams of uint32 words, the heads stream first and the conts stream
 * from chunk cont_base on (chunk c = words 64c..64c+63; group g's 4 words at 64c+4g; group g =
 * lanes 2g, 2g+1 of a warp, 32 B each of a 64-B row slice; pair q, half h sits in group
 * 4(q>>1) + (q&1) + 2h).  warp_info[nwarps*3] = {items, first head chunk, first cont chunk} per
 * consumer warp.  A slot is an 11-bit tile row (data m -> m, check i -> kpad+i, padding ->
 * zero_even or zero_even+1); a slot word packs two slots as a | b << 21.  An item's head chunk
 * holds, per group, word 0 = row | ctrl << 16 (ctrl = L | pair-split << 14 | warp-split << 15;
 * row 0xFFFF = no output) and slots 0..5 in words 1..3 (word 1 bit 11: the group's pair is a
 * pair-split); slots 6..L-1 follow in the conts stream, 8 per chunk.  In every step groups g and
 * g^2 read rows of opposite parity (shared-memory bank rule).  FS_EUNSUPPORTED when the graph is
 * not SMEM-eligible.                                                                         */
/* The fixed-size LT edge windows of the GLOBAL window kernel (host views, owned by g): window w
 * (w < *count) covers the LT rows [hdr[2w], hdr[2w+2]) (the last window ends at n); hdr[2w+1] =
 * its batches of 4 edges; its *entries edge slots ent[w * *entries ...] hold the rows' column
 * indices in row order, bit 31 set on each row's last edge, preceded by (4 - edges % 4) % 4
 * padding slots with bit 30 set (kernel skips them); the rest of the slots are 0.  Windows hold
 * at most 12 rows (FSB_WIN_ROWS) and 96 edge slots.  FS_EUNSUPPORTED when the graph has no
 * windows (a row of more than 93 edges).                                                    */
FSB_API fs_status fs_graph_windows(const fs_graph *g, const uint32_t **hdr, const uint32_t **ent,
                                   uint32_t *count, uint32_t *entries);

FSB_API fs_status fs_graph_schedule(const fs_graph *g, const uint32_t **words, uint64_t *nwords,
                                    uint32_t *cont_base, const uint32_t **warp_info, uint32_t *nwarps,
                                    uint32_t *kpad, uint32_t *zero_even);

/* ---------------------------------------------------------------- decoder
 * Decoding is split like the encoder: a graph-only plan on the host, then data-parallel XOR on
 * the GPU.  The plan follows Alg 5 (DPG): equations are the received LT rows
 * (Y_j = XOR of its neighbours) and the p precode checks (0 = XOR of P(i) and C_i; "BP at most
 * twice"); at level L every equation with exactly one unknown left recovers it, one
 * equation per unknown -- the lowest-degree one (ties: lowest index, LT rows
 * before checks) -- so a level's rows are independent.  The recovered set is the
 * peeling closure of Alg 1; unknowns in a stopping set stay unrecovered (the
 * paper's BP returns them as F).                                                             */
typedef struct fs_decode_plan fs_decode_plan;  /* opaque, immutable after creation */

typedef struct {
  uint32_t K;                /* intermediate symbols k+p                                        */
  uint32_t n;                /* coded symbols                                                   */
  uint32_t received;         /* received coded symbols                                          */
  uint32_t recovered;        /* intermediate symbols the plan recovers                          */
  uint32_t recovered_data;   /* ... of them data symbols (index < k)                            */
  uint32_t levels;           /* DPG levels (GPU launches per fs_decode)                         */
  uint32_t rows;             /* rows of the plan (= recovered)                                  */
  uint32_t max_level_rows;   /* largest level                                                   */
  uint64_t xor_sources;      /* total sources over all rows (XOR work per byte column)          */
  uint32_t eliminated;       /* symbols recovered after peeling stalled (FS_DECODE_ELIMINATE)   */
  uint32_t elim_skipped;     /* reserved (0)                                                    */
  uint32_t inactivated;      /* symbols inactivated by the completion phase                     */
  uint32_t work_rows;        /* device workspace rows per stripe (t bytes each, library-owned)  */
} fs_decode_info;

/* fs_decode_plan_create flag: complete the decode where peeling stalls, by inactivation decoding
 * (host plan, GPU rows): inactivate a few unknowns, keep peeling with them carried symbolically,
 * solve the small GF(2) system the unused equations give for them (Gauss-Jordan on the host), then
 * fix up every symbol that depended on them.  Recovers exactly the symbols the received equations
 * determine (state 2 for those peeling alone did not reach).  Rows of symbols that stay
 * unrecovered may then hold partial values.  fs_decode allocates the plan's workspace
 * (work_rows x t x stripes bytes) on first use.  Not in the paper (its decoder is BP only,
 * PAPER.md:113-134): SURVEY.md §8(f) NEXT-1's "inactivation / GF(2) fallback".              */
#define FS_DECODE_ELIMINATE 2u

/* Build the plan for graph g and the received set: received[j] != 0 iff coded symbol j is
 * available (n bytes, host).  flags: FS_GRAPH_HOST_ONLY = no device copy (fs_decode then
 * returns FS_EUNSUPPORTED); FS_DECODE_ELIMINATE = finish with GF(2) elimination (above).
 * FS_EINVAL on NULL arguments or unknown flags.                                             */
FSB_API fs_status fs_decode_plan_create(const fs_graph *g, const uint8_t *received, uint32_t flags,
                                        fs_decode_plan **out);
FSB_API fs_status fs_decode_plan_info(const fs_decode_plan *plan, fs_decode_info *info);
/* Host views owned by the plan: state[K] (1 = recovered by peeling, 2 = by elimination,
 * 0 = not recovered), level_of[K] (level, -1). */
FSB_API fs_status fs_decode_plan_state(const fs_decode_plan *plan, const uint8_t **state,
                                       const int32_t **level_of);
/* Run the plan on num_stripes stripes: d_coded = coded symbols (row j at d_coded + s*coded_stride
 * + j*t; rows not received are never read), d_inter = output intermediate symbols (row m at
 * d_inter + s*inter_stride + m*t; rows the plan recovers are written, the others untouched;
 * data symbols are rows 0..k-1).  Strides multiples of 16 and >= n*t, (k+p)*t.  One launch per
 * level on `stream`.                                                                          */
FSB_API fs_status fs_decode(const fs_decode_plan *plan, uint32_t num_stripes, const uint8_t *d_coded,
                            uint64_t coded_stride, uint8_t *d_inter, uint64_t inter_stride, void *stream);
FSB_API void fs_decode_plan_free(fs_decode_plan *plan);  /* NULL-safe */

/* ------------------------------------------------ repair, update, degraded read (NEXT-3)
 * Check #2 / Check #3 local sets from Algorithm 4, CGA,
 * run on the host over B = the LT generator (K x n; the paper's k is our K = k+p, reading R19).
 * A weight-0 column j of CGA's B gives a Group #3 set {C_s : l_{s,j} = 1} (coded symbols whose
 * XOR is zero); a weight-1 column (symbol x) a Group #2 set: I_x = XOR of its coded symbols.
 * Optional derived Group #3 sets: FS_CHECKS_M1 = degree-one coded nodes
 * (G_x setXOR {j}), FS_CHECKS_M2 = check #1 groups (setXOR of the members' G_x, Eq 4).  The sets
 * are serialised in the <filename>_check.data format: Group #3 as
 * [0, deg, c_1..c_deg], Group #2 as [1, x, deg, c_1..c_deg], smallest cardinality first
 * (ties by CGA column, derived sets after, reading R20).  CGA is a heuristic: it
 * may stop before every column has weight <= 1 (the info reports how far it got).          */
#define FS_CHECKS_M1 1u
#define FS_CHECKS_M2 2u

typedef struct fs_checks fs_checks;  /* opaque, immutable after creation */

typedef struct {
  uint32_t sweeps;           /* passes of CGA's while loop                                      */
  uint32_t zero_columns;     /* weight-0 columns at exit (the loop's target is n - K)           */
  uint32_t weight1_columns;  /* weight-1 columns at exit                                        */
  uint32_t group2;           /* Group #2 sets in the data                                       */
  uint32_t group3;           /* Group #3 sets in the data (incl. derived)                       */
  uint32_t derived;          /* derived Group #3 sets (FS_CHECKS_M1 / _M2)                      */
  uint64_t len;              /* int32 entries of the check data                                 */
} fs_checks_info;

/* Run CGA on g's LT graph and build the check data.  flags: FS_CHECKS_M1 | FS_CHECKS_M2.
 * Host only, deterministic.  FS_EINVAL on NULL arguments or unknown flags.                    */
FSB_API fs_status fs_checks_create(const fs_graph *g, uint32_t flags, fs_checks **out);
/* Adopt check data produced elsewhere (e.g. by an earlier graph, for an update): validated
 * against g (flags 0/1, sizes >= 1, coded indices < n, symbols < K); copied.  FS_EINVAL if not. */
FSB_API fs_status fs_checks_from_data(const fs_graph *g, const int32_t *data, uint64_t len, fs_checks **out);
/* Host view of the check data (owned by c, valid until fs_checks_free). */
FSB_API fs_status fs_checks_data(const fs_checks *c, const int32_t **data, uint64_t *len);
FSB_API fs_status fs_checks_info_get(const fs_checks *c, fs_checks_info *info);
FSB_API void fs_checks_free(fs_checks *c);  /* NULL-safe */

/* Repair plan (reading R21) for graph g (its LT rows are the base
 * graph; for an update, g is the extended graph and c the check data of the original code):
 * unknowns = the erased coded symbols (erased[j] != 0, n bytes, host).  Rounds of
 *   A: each Group #3 set, in order, with exactly one unknown member repairs it (XOR of the rest);
 *   B: each unknown coded symbol j, ascending, whose every neighbour x has a Group #2 set with
 *      all members known: C_j = XOR over x of XOR(G_x)   (the Eq 4 setXOR construction)
 * repeat while either resolves something; then each of the nwant wanted intermediate symbols
 * want[] (degraded read) from its first Group #2 set with all members known.
 * Rows run in levels (1 + max level of the sources); the unresolved remain (decode + encode
 * rebuilds those).  flags: FS_GRAPH_HOST_ONLY = no device copy.                              */
typedef struct fs_repair_plan fs_repair_plan;  /* opaque, immutable after creation */

typedef struct {
  uint32_t erased;           /* erased coded symbols                                            */
  uint32_t repaired;         /* ... the plan rebuilds                                           */
  uint32_t unrepaired;       /* ... it cannot (no usable local set)                             */
  uint32_t want_missing;     /* wanted intermediate symbols without a usable Group #2 set       */
  uint32_t levels;           /* GPU launches per fs_repair                                      */
  uint32_t rows;             /* plan rows (repaired + wanted rows)                              */
  uint64_t xor_sources;      /* total sources over all rows                                     */
} fs_repair_info;

FSB_API fs_status fs_repair_plan_create(const fs_graph *g, const fs_checks *c, const uint8_t *erased,
                                        const uint32_t *want, uint32_t nwant, uint32_t flags,
                                        fs_repair_plan **out);
FSB_API fs_status fs_repair_plan_info(const fs_repair_plan *plan, fs_repair_info *info);
/* Host views of the plan rows: level_ptr[levels+1], target[rows] (bit 30 set: coded symbol,
 * clear: intermediate symbol), src_ptr[rows+1], src[...] (coded indices | bit 30, bit 31 marks a
 * row's last source).  Owned by the plan.                                                    */
FSB_API fs_status fs_repair_plan_rows(const fs_repair_plan *plan, const uint32_t **level_ptr,
                                      uint32_t *levels, const int32_t **target, const int32_t **src_ptr,
                                      const uint32_t **src);
/* Run the plan on num_stripes stripes, in place: repaired rows are written into d_coded (row j
 * at d_coded + s*coded_stride + j*t; erased rows are never read before they are written);
 * wanted intermediate rows into d_inter (row x at d_inter + s*inter_stride + x*t), which may
 * be NULL when the plan has none.  Strides multiples of 16, >= n*t and (k+p)*t.  One launch
 * per level on `stream`.                                                                     */
FSB_API fs_status fs_repair(const fs_repair_plan *plan, uint32_t num_stripes, uint8_t *d_coded,
                            uint64_t coded_stride, uint8_t *d_inter, uint64_t inter_stride, void *stream);
FSB_API void fs_repair_plan_free(fs_repair_plan *plan);  /* NULL-safe */

/* Update: the code extended by extra_files output files.  With s =
 * max(files, 1), the new graph has n' = n + extra_files * n/s rows and files' = s + extra_files;
 * file i's rows come from stream seed + i (R17), so rows 0..n-1 are exactly g's and the new
 * rows n..n'-1 are drawn from fresh streams.  Their symbols are computed with fs_encode (row
 * range [n, n')) from the data, or, with the data not stored, by fs_repair on the new graph
 * with the original code's check data and rows n..n'-1 marked erased.  flags as for
 * fs_graph_create.  FS_EINVAL if extra_files == 0 or n' overflows.                           */
FSB_API fs_status fs_graph_extend(const fs_graph *g, uint32_t extra_files, uint32_t flags, fs_graph **out);

/* Profiling aid (only meaningful when the process runs with FSB_DEBUG=2): copies out and clears
 * n <= 64 counters of the SMEM kernel: for consumer warp w, [2w] = cycles spent waiting for tiles,
 * [2w+1] = total cycles, each summed over all CTAs since the last call.                    */
FSB_API fs_status fs_debug_counters(uint64_t *out, uint32_t n);

/* Number of kernel launches the last successful fs_encode / fs_encode_stripes on this
 * thread enqueued (for launch accounting in benchmarks).                                 */
FSB_API uint32_t fs_last_launch_count(void);

/* Frees everything g owns (device memory on its device).  NULL-safe.                     */
FSB_API void fs_free(fs_graph *g);

/* Thread-local description of the last error ("" if none). */
FSB_API const char *fs_last_error(void);

/* Library version string. */
FSB_API const char *fs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FSB_H_ */
