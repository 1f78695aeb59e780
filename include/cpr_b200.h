/*
 * cpr_b200.h — C ABI of the B200-native CPR-GMRES SOLVE path.
 *
 * The reference (cprkit, pure Python) has no FFI: its boundary is the Python
 * API.  This header is the C-ABI the Python drop-in
 * (paper_2201_01970_b200) binds through ctypes; each entry point names the
 * reference function it replaces (src/X.py:N = cprkit/X.py line N).
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device memory
 *    (owned by the caller, e.g. torch tensors); everything else is host.
 *  - `stream` is a cudaStream_t passed as void*; all device calls are
 *    stream-ordered and asynchronous unless stated.
 *  - Return value: CPRB_OK or an error code; cprb_last_error() gives the
 *    message (thread-local).  The Python layer maps codes to the reference's
 *    exception types.
 *  - Index types: setup uses int64 (the reference's index dtype); device
 *    layouts use int32 (max nnz at the 26.9M-DOF config is 6.3e7 blocks).
 */
#ifndef CPR_B200_H
#define CPR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CPRB_OK = 0,
  CPRB_EINVAL = 1,     /* ValueError            (e.g. dimension mismatch) */
  CPRB_ENONFINITE = 2, /* FloatingPointError    (src/cpr.py:248,274,307) */
  CPRB_ESINGULAR = 3,  /* numpy.linalg.LinAlgError (src/ilu.py:140,147; src/smoothers.py:89) */
  CPRB_EDEVICE = 4,    /* RuntimeError: CUDA failure */
  CPRB_ERUNTIME = 5,   /* RuntimeError (src/amg.py:172) */
  CPRB_EUNSUPPORTED = 6
};

const char* cprb_last_error(void);
int cprb_version(void);

/* ======================= host setup (SETUP phase) ======================= */

/* src/coloring.py:79-114  S(A,theta): S_ij iff i!=j and |a_ij| > theta*sum_k|a_ik|
 * (row sum in numpy reduceat order).  s_ptr[n+1], s_cols[capacity nnz]. */
int cprb_strong_connections(int64_t n, const int64_t* ptr, const int64_t* cols,
                            const double* vals, double theta, int64_t* s_ptr,
                            int64_t* s_cols);

/* src/coloring.py:238-256 (+ vertices_splitting :171-235)  greedy colour
 * groups on S ∪ S^T.  perm[n] = concatenated ascending groups;
 * group_sizes[capacity n]; *ncolors = number of groups. */
int cprb_vertices_grouping(int64_t n, const int64_t* s_ptr, const int64_t* s_cols,
                           int64_t* perm, int64_t* group_sizes, int64_t* ncolors);

/* src/amg.py:89-119  greedy pairwise aggregation (NPAIR). agg[n], *n_agg. */
int cprb_pairwise_aggregate(int64_t n, const int64_t* ptr, const int64_t* cols,
                            const double* vals, double theta_amg, int64_t* agg,
                            int64_t* n_agg);

/* src/amg.py:127-132  Galerkin A_c = P^T A P for piecewise-constant P,
 * duplicate sums in stable-lexsort + reduceat order.  Outputs have capacity
 * nnz(A); c_ptr[n_agg+1]; *c_nnz. */
int cprb_galerkin(int64_t n, const int64_t* ptr, const int64_t* cols, const double* vals,
                  const int64_t* agg, int64_t n_agg, int64_t* c_ptr, int64_t* c_cols,
                  double* c_vals, int64_t* c_nnz);

/* src/amg.py:135-140 */
int cprb_is_symmetric(int64_t n, const int64_t* ptr, const int64_t* cols, const double* vals,
                      double tol, int32_t* out);

/* src/ilu.py:150-193  BILU(0), IKJ on the pattern; `vals` (nnz*b*b) is
 * overwritten with the factors, uinv[n*b*b] = inverted pivots (Gauss-Jordan,
 * src/sparse.py:372-396).  Perturbed pivots (src/ilu.py:134-147) are listed in
 * perturbed[capacity n]; *n_perturbed.  CPRB_ESINGULAR names the row. */
int cprb_bilu0_factorize(int64_t n, int32_t b, const int64_t* ptr, const int64_t* cols,
                         double* vals, double* uinv, int64_t* perturbed,
                         int64_t* n_perturbed);

/* src/ilu.py:38-59  level[i] (1-based) of a triangular pattern; *nlevels. */
int cprb_level_schedule(int64_t n, const int64_t* ptr, const int64_t* cols,
                        int64_t* level, int64_t* nlevels);

/* src/ilu.py:38-59 applied to the strict lower part of A's own pattern (the
 * BILU(0) factorization's row dependencies).  level[n], *nlevels. */
int cprb_lower_level_schedule(int64_t n, const int64_t* ptr, const int64_t* cols,
                              int64_t* level, int64_t* nlevels);

/* src/smoothers.py:257-271  colour-permuted split of a scalar matrix: row
 * pr = inv[r] holds (inv[c], a_rc), c != r, in ascending inv[c]; diag[pr] =
 * a_rr (CPRB_ESINGULAR names the first zero diagonal, permuted index). */
int cprb_scalar_split(int64_t n, const int64_t* ptr, const int64_t* cols, const double* vals,
                      const int64_t* perm, const int64_t* inv, int64_t* off_ptr,
                      int64_t* off_cols, double* off_vals, double* diag);

/* Host SELL-32 fills for the device layouts (cprb_sell): from per-lane
 * entry lists, or from the rows of a scalar CSR (lane_src[l] = row, -1 =
 * padding; columns renumbered through colmap when non-NULL).  Outputs are
 * zero-initialised by the caller and sized by slice_ptr[L/32]. */
int cprb_sell_fill_lanes(int64_t L, const int64_t* lane_ptr, const int64_t* slice_ptr,
                         const int64_t* ent_cols, const double* ent_vals, int32_t bs,
                         int32_t* out_cols, double* out_vals);
int cprb_sell_fill_rows(int64_t L, const int64_t* lane_src, const int64_t* slice_ptr,
                        const int64_t* ptr, const int64_t* cols, const double* vals,
                        const int64_t* colmap, int32_t* out_cols, double* out_vals);

/* Structured 7-point grid test for the stencil BILU plan: returns 1 and
 * dims[3] = {nx, ny, nz} when every row's block columns are exactly the
 * in-range neighbours of a natural-ordered grid (nx, ny, nz >= 2), else 0. */
int cprb_detect_stencil(int64_t n, const int64_t* ptr, const int64_t* cols, int64_t* dims);

/* src/mmio.py:36-95  body of a MatrixMarket coordinate file (after the
 * header line).  info[12] out: nrows, ncols, nnz, block_size sidecar (-1 =
 * none), entries read, error code (0 ok; 1 sidecar, 2/3 size line, 4 no size
 * line, 5 entry, 6 index range (info[7..8] = i, j), 7 too many entries,
 * 8 count mismatch, 9 token outside the fast grammar), error line, -, -,
 * total lines.  rows/cols/vals/linenos (capacity nnz) may be NULL to read
 * the size line only.  Entries are 0-based. */
int cprb_mm_read_coord(const char* path, int64_t* rows, int64_t* cols, double* vals,
                       int64_t* linenos, int64_t* info);
/* src/mmio.py:149-160  append "i j v" lines (1-based, %.17g). */
int cprb_mm_write_entries(const char* path, int64_t n, const int64_t* rows, const int64_t* cols,
                          const double* vals);

/* coarsest level (replaces scipy lu_factor/lu_solve, src/amg.py:170-173,
 * :248-249): dense inverse via LU with partial pivoting; a: n*n row-major. */
int cprb_dense_inverse(int64_t n, const double* a, double* inv);

/* src/sparse.py:372-396 batched 3x3/bxb Gauss-Jordan inverse (bitwise). */
int cprb_invert_small_blocks(int64_t m, int32_t b, const double* blocks, double* out);

/* ===================== device layouts (SOLVE phase) ===================== */

/* SELL-32 sliced-ELL storage.  Slice s owns 32 lanes; lane l of slice s maps
 * to row lane_row[s*32+l] (-1 = padding).  Entry m of that lane is at
 * e = slice_ptr[s] + m*32 + l:  cols[e];  scalar value vals[e];  b x b block
 * value (r,c) at vals[(slice_ptr[s] + m*32)*b*b + (r*b+c)*32 + l].
 * Entries of a row keep the reference's summation order. */
typedef struct cprb_sell {
  int32_t nslices;
  int32_t nrows;
  const int64_t* slice_ptr;   /* dev, nslices+1 (entry units) */
  const int32_t* lane_row;    /* dev, nslices*32 */
  const int32_t* lane_len;    /* dev, nslices*32 */
  const int32_t* lane_len_lo; /* dev|NULL: entries with col < colour start */
  const int32_t* cols;        /* dev */
  const double* vals;         /* dev */
  const int32_t* agg_out;     /* dev|NULL: restriction output index per lane pair */
} cprb_sell;

/* One smoothed AMG level (src/amg.py:68-74 AmgLevel), in colour-permuted
 * order.  HOST arrays: colour bounds. */
typedef struct cprb_amg_level {
  int32_t n;
  int32_t ncolors;
  const int32_t* color_slices; /* host, ncolors+1 (slice bounds in `smoother`) */
  const int32_t* color_rows;   /* host, ncolors+1 (row bounds, permuted)        */
  const uint8_t* color_snapshot; /* host, ncolors: 1 = intra-colour couplings  */
  cprb_sell smoother;          /* off-diagonals, ascending permuted columns     */
  const double* diag;          /* dev, n */
  cprb_sell restrict_op;       /* rows grouped by aggregate (lane pairs), original column order */
  const int32_t* aggp;         /* dev, n: coarse (permuted) index of each row   */
  double* b;                   /* dev work, n */
  double* x;                   /* dev work, n */
  double* tmp;                 /* dev work, n (snapshot sweeps) */
  const int32_t* color_width;  /* host|NULL, 2*ncolors: max lane_len, max lane_len_lo per colour */
  int32_t restrict_width;      /* max row length of restrict_op (0 = unknown) */
  int32_t pad_;
} cprb_amg_level;

typedef struct cprb_amg {
  int32_t nlevels;                  /* total, including the coarsest */
  const cprb_amg_level* levels;     /* host array, nlevels-1 entries  */
  int32_t n_coarse;
  const double* coarse_inv;         /* dev, n_coarse^2 row-major */
  double* coarse_b;                 /* dev work */
  double* coarse_x;                 /* dev work */
  const int32_t* perm0;             /* dev, n0: level-0 permuted row -> fine index */
  int32_t in_stride;                /* residual stride of the level-0 input (b of BSR, 1 scalar) */
  int32_t cycle;                    /* 0 = V, 1 = K */
  int32_t use_fcg;                  /* K-cycle Krylov flavour */
  void* kwork;                       /* K-cycle plan (cprb_kcycle_create) or NULL; used when cycle = 1 */
  int64_t kwork_len;
  /* persistent single-CTA V-cycle tail (csrc/vtail.cu): levels >= tail_start
   * and the coarse solve in one launch, vectors in shared memory, static
   * records streamed by TMA; tail_start >= nlevels-1 disables it. */
  int32_t tail_start;
  int32_t tail_nphases;
  int32_t tail_nchunks;
  int32_t tail_slot;                /* ring slot bytes (multiple of 16) */
  int32_t tail_smem;                /* dynamic shared memory bytes of the launch */
  int32_t tail_vec_len;             /* doubles of the shared-memory vector region */
  const int32_t* tail_phases;       /* dev, (nphases+1) x {type, level, colour|zg, first chunk} */
  const int32_t* tail_chunks;       /* dev, nchunks x {phase, 16-byte offset, bytes, rows} */
  const uint8_t* tail_stream;       /* dev, packed chunk records */
  const int32_t* tail_vec;          /* dev, 2*nlevels: shared-memory offsets of b_l, x_l */
  int64_t tail_stream_bytes;        /* bytes of tail_stream (L2 persistence window) */
} cprb_amg;

/* Chunked-wavefront plan of one triangular factor (csrc/wave.cu).  Rows are
 * cut into contiguous chunks of one dependency bandwidth; inside a chunk rows
 * are grouped into level "steps" (<= 64 rows).  Each step is one contiguous,
 * 16-byte aligned block of `stream`:
 *   int32 rows[Wp], lens[Wp], aux[Wp], codes[K][Wp];
 *   f64 vals[K][b*b][Wp]; (upper factor) f64 uinv[b*b][Wp]
 * with Wp = round_up(w, 4); a code < 0 names a shared-memory ring slot
 * (-code-1), otherwise the dependency's row.  The step's right-hand side is
 * rhs[rhs_off[k] ...] (w*b doubles, 16-byte aligned). */
typedef struct cprb_wave {
  int32_t nchunks;
  int32_t nsteps;
  int32_t stage_max;           /* max step_bytes (multiple of 16) */
  int32_t rhs_max;             /* max rhs_bytes (multiple of 16) */
  const int32_t* chunk_step;   /* dev, nchunks+1 */
  const int64_t* step_off;     /* dev, byte offsets into stream */
  const int32_t* step_bytes;   /* dev */
  const int32_t* step_w;       /* dev */
  const int32_t* step_k;       /* dev */
  const int64_t* rhs_off;      /* dev, double offsets into the rhs vector */
  const int32_t* rhs_bytes;    /* dev */
  const uint8_t* stream;       /* dev */
  int32_t max_chunk_steps;     /* longest chunk (steps); <= 320: metadata staged in smem */
  int32_t pad_;
} cprb_wave;

/* Structured-grid ("stencil") BILU(0) plan: the factors of a natural-ordered
 * nx x ny x nz 7-point grid (exactly the in-range neighbours, so ILU(0)'s L
 * and U patterns are the -z,-y,-x / +x,+y,+z stencils), stored per xy-plane
 * in anti-diagonal order (d = ix + iy).  Row (ix, iy, iz) sits at position
 * iz*P + doff[d] + (ix - lo(d)) (diagonal blocks padded to an even width:
 * 16-byte TMA granules); its record is contiguous: L 27 doubles, fields
 * m*9 + e (m: 0 -z, 1 -y, 2 -x; e = r*3 + c), U 37 doubles, fields m*9 + e
 * (m: 0 +x, 1 +y, 2 +z), the 9 entries of inv(U_ii), one pad word. */
typedef struct cprb_stencil {
  int32_t nx, ny, nz;          /* grid (x fastest) */
  int32_t S;                   /* x-segments of 32 lanes (ceil(nx / 32) <= 4) */
  int32_t D;                   /* anti-diagonals per plane (nx + ny - 1) */
  int32_t P;                   /* padded rows per plane (doff[D]) */
  const int32_t* doff;         /* dev, D + 1 padded diagonal offsets */
  const double* lrec;          /* dev, nz * P * 27 */
  const double* urec;          /* dev, nz * P * 37 */
} cprb_stencil;

typedef struct cprb_bilu {
  int32_t n;                   /* block rows */
  int32_t b;                   /* block size (1 or 3) */
  cprb_sell L;                 /* strict lower blocks; lanes in L-level order */
  cprb_sell U;                 /* strict upper blocks; lanes in U-level order */
  const double* uinv;          /* dev, U lane layout: [(s*b*b + e)*32 + l] */
  int32_t* tickets;            /* dev, 4 ints (dynamic warp / chunk ordering) */
  int32_t use_wave;            /* 1: chunked-wavefront kernels (Lw/Uw); 2: stencil plan (St) */
  cprb_wave Lw;
  cprb_wave Uw;
  const int32_t* l_slot;       /* dev, n: rhs slot of each row in the L plan */
  double* rhs_l;               /* dev work: rhs in L step order */
  double* rhs_u;               /* dev work: z in U step order (U solve input) */
  const int32_t* u_slot;       /* dev, n: rhs slot of each row in the U plan */
  double* zl_step;             /* dev work: z in L step order (L output, sentinel-polled) */
  double* y_step;              /* dev work: y in U step order (U output, sentinel-polled) */
  int64_t len_l;               /* doubles in rhs_l / zl_step */
  int64_t len_u;               /* doubles in rhs_u / y_step */
  cprb_stencil St;             /* use_wave == 2: l_slot == u_slot = 3 * stencil position */
} cprb_bilu;

typedef struct cprb_cpr {
  int32_t nb;                  /* block rows */
  int32_t b;                   /* block size */
  cprb_sell A;                 /* build-time matrix (stage-2 residual) */
  cprb_amg amg;
  cprb_bilu bilu;
  double* zp;                  /* dev work, nb: pressure correction, natural order */
  double* r2;                  /* dev work, nb*b */
  double* zl;                  /* dev work, nb*b (L-solve, sentinel polled) */
  double* y;                   /* dev work, nb*b (U-solve, sentinel polled) */
} cprb_cpr;

/* ============================ device kernels ============================ */

/* SETUP on the device.  src/ilu.py:150-193 BILU(0) of a 3x3-block matrix in
 * place on A's pattern (dev ptr/cols int64, vals n_blocks*9), uinv[n*9] =
 * inverted pivots; rows are processed level by level (level_rows: dev int32,
 * rows grouped by cprb_lower_level_schedule level; level_ptr: HOST int64,
 * nlevels+1).  err: dev int32[4] -> {lowest zero-pivot row, lowest row
 * without a diagonal block (INT32_MAX = none), number of perturbed pivots};
 * perturbed: dev int64[n] (unordered).  Bitwise the host factorization. */
int cprb_bilu0_factorize_device(int64_t n, int32_t b, const int64_t* ptr, const int64_t* cols,
                                double* vals, double* uinv, const int32_t* level_rows,
                                const int64_t* level_ptr, int64_t nlevels, int32_t* err,
                                int64_t* perturbed, void* stream);
/* Factored CSR (A's pattern) -> stencil records (cprb_stencil lrec/urec,
 * zero-initialised by the caller) and the per-row rhs slot (3 * position). */
int cprb_stencil_pack(int64_t n, int32_t nx, int32_t ny, int32_t P, const int32_t* doff,
                      const int64_t* ptr, const int64_t* cols, const double* vals,
                      const double* uinv, double* lrec, double* urec, int32_t* slot,
                      void* stream);
/* src/problems.py:113-155 on the device (nx*ny*nz cells, 3x3 blocks):
 * row counts, then the rows (int64 block columns ascending, 9 values per
 * block) given the host-drawn perm = exp(logk), conv_scale and couple[n*6]. */
int cprb_gen_row_counts(int64_t nx, int64_t ny, int64_t nz, int64_t* cnt, void* stream);
int cprb_gen_assemble(int64_t nx, int64_t ny, int64_t nz, double drift, const double* perm,
                      const double* conv_scale, const double* couple, const int64_t* row_ptr,
                      int64_t* cols, double* vals, void* stream);

/* src/sparse.py:335-351  y = A x (BSR via the expanded-row order).  flag
 * (dev|NULL) is set to 1 when any y is non-finite. */
int cprb_spmv(const cprb_sell* A, int32_t b, const double* x, double* y, int32_t* flag,
              void* stream);
/* r = rhs - A x  (src/cpr.py:246, :306) */
int cprb_residual(const cprb_sell* A, int32_t b, const double* rhs, const double* x,
                  double* r, int32_t* flag, void* stream);

/* src/smoothers.py:273-318  one PGS-SCM pass over a level (permuted vectors).
 * direction 0 forward / 1 backward; zero_guess: x is treated as 0. */
int cprb_pgs_scm_pass(const cprb_amg_level* lvl, const double* b, double* x, int32_t direction,
                      int32_t zero_guess, void* stream);

/* src/amg.py:228-267  z = amg_cycle(h, r); r strided by h->in_stride. */
int cprb_amg_cycle(const cprb_amg* h, const double* r, double* z, void* stream);

/* K-cycle building blocks (the K-cycle recursion, src/amg.py:177-225,
 * :256-263, is driven by the host layer with these device steps). */
int cprb_coarse_solve(const cprb_amg* h, const double* b, double* x, void* stream);
int cprb_resid_restrict(const cprb_amg_level* lvl, const double* b, const double* x, double* bc,
                        void* stream);
int cprb_prolong(const cprb_amg_level* lvl, const double* xc, double* x, void* stream);

/* src/amg.py:177-196, :245-267  device K-cycle plan (FCG flavour): workspace
 * for every level and the level matrices in permuted row order with the
 * reference's column order (level_spmv: host array of nlevels-1 descriptors;
 * entry 0 unused).  With h->kwork = plan and h->cycle = 1, cprb_amg_cycle /
 * cprb_cpr_apply run the K-cycle without host synchronisation. */
int cprb_kcycle_create(const cprb_amg* h, const cprb_sell* level_spmv, int32_t pre_sweeps,
                       int32_t post_sweeps, void** plan);
int cprb_kcycle_destroy(void* plan);
/* K-cycle coarse correction from level l >= 1 (src/amg.py:256-263) on
 * natural-order vectors (perm: level-permuted row -> natural index). */
int cprb_kcycle_correction(const cprb_amg* h, int32_t l, const int32_t* perm, const double* rhs,
                           double* out, void* stream);

/* src/ilu.py:196-223  z = U^{-1} L^{-1} r (level-ordered, sync-free). */
int cprb_bilu_apply(const cprb_bilu* F, const double* r, double* z, double* work_l,
                    void* stream);

/* Diagnostic: record per-step completion times of the wave solves into
 * dev_log ([2][256 chunks][512 steps] uint64, %globaltimer); NULL = off. */
int cprb_wave_set_log(uint64_t* dev_log);
/* Diagnostic: per-plane timeline of the stencil BILU solves ([2][1024 planes]
 * x 8 u64: start/end %globaltimer, cycles in TMA waits, cycles in plane
 * waits, total cycles, diagonals); NULL = off. */
int cprb_stencil_set_log(uint64_t* dev_log);
/* Diagnostic: persistent V-cycle tail timeline (consumer thread 0: start,
 * after the PDL wait, then the end of every phase; u64 %globaltimer). */
int cprb_vtail_set_log(uint64_t* dev_log);
/* Diagnostic: V-cycle kernel timeline ({kind, start, after-wait, end} u64 per
 * launch, %globaltimer, <= 4096 launches); resets the counter; NULL = off. */
int cprb_amg_set_log(uint64_t* dev_log);

/* src/cpr.py:178-186  z = B r (V-cycle pressure stage). */
int cprb_cpr_apply(const cprb_cpr* P, const double* r, double* z, void* stream);
/* Graph-replayed cprb_cpr_apply: one cached CUDA graph per (P, r, z). */
int cprb_graph_cache_create(void** out);
int cprb_graph_cache_destroy(void* cache);
int cprb_cpr_apply_graph(void* cache, const cprb_cpr* P, const double* r, double* z, void* stream);
int cprb_amg_cycle_graph(void* cache, const cprb_amg* h, const double* r, double* z, void* stream);
/* src/cpr.py:184-186  second half given zp already in P->zp. */
int cprb_cpr_finish(const cprb_cpr* P, const double* r, double* z, void* stream);

/* Deterministic reductions (fixed block partition + fixed tree).
 * partials: dev, >= CPRB_RED_BLOCKS doubles; ticket: dev int (zeroed once). */
#define CPRB_RED_BLOCKS 1184
int cprb_dot(int64_t n, const double* x, const double* y, double* out, double* partials,
             int32_t* ticket, void* stream);

/* *out = sqrt((x, x)) on the device (same reduction as cprb_dot, IEEE sqrt):
 * src/sparse.py:361-369 norm2 without a host round trip. */
int cprb_norm2(int64_t n, const double* x, double* out, double* partials, int32_t* ticket,
               void* stream);

/* src/cpr.py:276-284  Arnoldi MGS for column j: for i<=j: H[i]=(w,V_i),
 * w -= H[i] V_i; H[j+1] = ||w||; V_{j+1} = w / H[j+1] (if nonzero).
 * V: (j+2) rows of length n (row stride ldv); w is V_{j+1} (in place). */
int cprb_arnoldi_mgs(int64_t n, int32_t j, double* V, int64_t ldv, double* Hcol,
                     double* partials, int32_t* ticket, void* stream);

/* u = sum_i y[i] V_i  (src/cpr.py:304), y: dev, k entries */
int cprb_gemv_t(int64_t n, int32_t k, const double* V, int64_t ldv, const double* y, double* u,
                void* stream);
/* out = x + s (elementwise, src/cpr.py:305) */
int cprb_add(int64_t n, const double* x, const double* s, double* out, void* stream);
/* out = alpha * x + y  (src/sparse.py:354-358; also the FCG updates of src/amg.py:188-194) */
int cprb_axpy(int64_t n, double alpha, const double* x, const double* y, double* out, void* stream);
/* out = x / h (host scalar; src/amg.py:204 rhs / beta) */
int cprb_div_host(int64_t n, const double* x, double h, double* out, void* stream);
/* out = x / (*h_dev)  (src/cpr.py:262 V[0] = r / beta) */
int cprb_div_scalar(int64_t n, const double* x, const double* h_dev, double* out, void* stream);

/* src/cpr.py:231-316  restarted right-preconditioned GMRES driven in C++
 * (for hosts without Python): solves A x = rhs from the initial guess in x
 * (dev, overwritten by the solution).  P: CPR preconditioner or NULL;
 * graphs: cprb_graph_cache_create cache or NULL (plain launches).
 * work: dev doubles, >= (m+1)*n + 3*n + 2*m + 3 + CPRB_RED_BLOCKS;
 * iwork: dev int32[4].  result[4] out (host): outer, inner, converged (0/1),
 * rel_residual.  Same steps and stopping rules as the Python driver; the
 * triangular solve is a plain back substitution (x agrees with the Python
 * driver to rounding); a zero Hessenberg pivot returns CPRB_EUNSUPPORTED. */
int cprb_gmres_solve(const cprb_sell* A, int32_t b, const cprb_cpr* P, void* graphs, int64_t n,
                     const double* rhs, double* x, int32_t m, int32_t max_restarts, double tol,
                     double* work, int32_t* iwork, double* result, void* stream);

/* Device SELL-32 packing of a (block) CSR matrix in natural row order
 * (uploads of new Jacobians, src/sparse.py:203-308 layout -> cprb_sell):
 * row_ptr/col_idx int64 and values (nnz*b*b) are device copies of the CSR
 * arrays; slice_ptr (host-computed widths) is on the device; cols/vals are
 * zero-filled outputs of slice_ptr[nslices] (x b*b) entries. */
int cprb_pack_bsr_sell(int64_t nrows, int32_t b, const int64_t* row_ptr, const int64_t* col_idx,
                       const double* values, const int64_t* slice_ptr, int32_t* cols,
                       double* vals, void* stream);

/* ---- slab-partitioned BILU (global wavefront, chunks cut at the slab
 * boundaries; each rank runs its own chunks and stores the rows another
 * rank reads (plan bit 29) into that rank's output array as well: peer_out,
 * NVLink peer memory, same offset).  Output arrays and right-hand sides are
 * per rank (explicit pointers); plan arrays come from F. */
int cprb_wave_solve_part(const cprb_bilu* F, int32_t upper, int32_t chunk0, int32_t nchunks,
                         const double* rhs_steps, double* out_step, double* peer_out,
                         int32_t* ticket, void* stream);
int cprb_l_to_u_rows(const cprb_bilu* F, int32_t row0, int32_t nrows, const double* zl_step,
                     double* rhs_u, void* stream);
int cprb_wave_combine_rows(const cprb_bilu* F, int32_t row0, int32_t nrows, const double* y_step,
                           const double* zp, double* z, void* stream);
int cprb_fill_sentinel_idx(int64_t n, int32_t b, const int32_t* idx, double* base, void* stream);
int cprb_stage2_residual_steps(const cprb_sell* A, const cprb_bilu* F, int32_t row0,
                               const double* zp, const double* r, double* rhs_l, double* zl_step,
                               double* y_step, void* stream);

/* ---- slab-partitioned solve (paper_2201_01970_b200/partition.py) ----
 * Each rank owns a contiguous range of block rows; operators read a column
 * window whose halo the host exchanges (NCCL over NVLink). */
/* src/cpr.py:185  r2 = r - A (Pi zp) (block column 0 only; zp one value per block column). */
int cprb_stage2_residual(const cprb_sell* A, int32_t b, const double* zp, const double* r,
                         double* r2, void* stream);
/* One colour of src/smoothers.py:273-318 (halo exchanged by the caller between colours). */
int cprb_pgs_scm_color(const cprb_amg_level* lvl, int32_t k, double* b, double* x,
                       int32_t zero_guess, const double* gsrc, int32_t gstride,
                       const int32_t* perm, double* sout, void* stream);
/* GPU-count-invariant reductions (src/sparse.py:361-369, src/cpr.py:276-284):
 * per fixed global segment of seg_len entries one partial of (w, vdot)
 * ((w, w) if vdot == NULL), after an optional MGS update w -= (*hprev) vprev;
 * then the fixed-order sum of nseg partials (map: global segment -> slot,
 * NULL = identity), square-rooted if sqrt_. */
int cprb_seg_partials(int64_t n, int64_t seg_len, double* w, const double* vprev,
                      const double* hprev, const double* vdot, double* partials, void* stream);
int cprb_seg_finish(int32_t nseg, const double* partials, const int32_t* map, double* out,
                    int32_t sqrt_, void* stream);
/* w /= *h unless *h == 0 (src/cpr.py:281-284). */
int cprb_div_if_nonzero(int64_t n, double* w, const double* h, void* stream);
/* dst[idx[i]] += src[i]  (cross-slab aggregates of np.bincount, src/amg.py:254-255). */
int cprb_scatter_add(int64_t n, const int32_t* idx, const double* src, double* dst, void* stream);
/* dst[i] = src[stride * idx[i]]  (halo packing; idx NULL = identity). */
int cprb_gather(int64_t n, const int32_t* idx, const double* src, int32_t stride, double* dst,
                void* stream);
/* padded all-gather [nranks][cap] -> packed; offs: device int64[nranks + 1]. */
int cprb_unpad(int32_t nranks, int64_t cap, const int64_t* offs, const double* src, double* dst,
               void* stream);
/* src/cpr.py:184-186  z = Pi zp + y  for ncells block rows of size b. */
int cprb_cpr_combine(int64_t ncells, int32_t b, const double* zp, const double* y, double* z,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CPR_B200_H */
