/*
 * hsseig_b200 — C ABI of the B200 (sm_100a) divide-and-conquer merge step.
 *
 * Drop-in for the merge-path functions of the reference package `hsseig`
 * (arXiv 1510.04591 reference, pkg/src/hsseig).  Every entry point takes
 * DEVICE pointers owned by the caller (PyTorch tensors in the Python host
 * layer), plain integer sizes and a cudaStream_t passed as `void *`.
 * Nothing here allocates or frees caller memory.  All arrays are float64,
 * C-contiguous (row-major) unless a leading dimension says otherwise.
 *
 * Calls are asynchronous on `stream`.  The return value reports argument
 * and launch errors only; numerical failures the reference raises as
 * exceptions are written to a caller-provided device status block and read
 * by the host once the stream is synchronised (see hsseig_status).
 */
#ifndef HSSEIG_B200_H
#define HSSEIG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return / status codes */
#define HSSEIG_OK 0
#define HSSEIG_ERR_ARG 1          /* ValueError */
#define HSSEIG_ERR_BRACKET 2      /* SecularConvergenceError, secular.py:25,172-179 */
#define HSSEIG_ERR_RADICAND 3     /* WeightRecomputationError, secular.py:29,226-230 */
#define HSSEIG_ERR_CUDA 4

/*
 * Device status block written by the kernels (int64 x 8):
 *   [0] total secular iterations     [1] first root with gamma<=0 (or k)
 *   [2] first root with mu<=0 (or k) [3] first bad Loewner radicand (or k)
 *   [4] HSS saturated-ID count       [5] max ID rank used (r_used)
 *   [6], [7] reserved
 */
typedef struct hsseig_status {
  int64_t v[8];
} hsseig_status;

/* Library identification (build check) and the number of kernels launched so far. */
const char *hsseig_version(void);
int64_t hsseig_launch_count(void);
/* Where the last HSSEIG_ERR_ARG of this thread came from ("invalid argument (file:line)"). */
const char *hsseig_last_error(void);
int hsseig_status_init(hsseig_status *status_dev, int64_t k, void *stream);

/*
 * (a1) All k secular roots with gap pairs.
 * Replaces secular_all (pkg/src/hsseig/_kernels.pyx:178-234) behind
 * solve_secular (pkg/src/hsseig/secular.py:159-180).
 * d: k strictly ascending poles; z: k nonzero weights; rho > 0.
 * lam/gamma/mu: k outputs; iters: k per-root iteration counts (int32).
 * work: >= 2*k + 64 doubles of device scratch, 16-byte aligned (packed poles).
 * status[0] += total iterations; status[1]/[2] = first bracket loss.
 */
int hsseig_secular(const double *d, const double *z, int64_t k, double rho, double *lam,
                   double *gamma, double *mu, int32_t *iters, double *work,
                   hsseig_status *status, void *stream);
/* Roots [ibeg, iend) only (multi-GPU index shard); outputs hold iend - ibeg entries. */
int hsseig_secular_part(const double *d, const double *z, int64_t k, double rho, int64_t ibeg,
                        int64_t iend, double *lam, double *gamma, double *mu, int32_t *iters,
                        double *work, hsseig_status *status, void *stream);

/*
 * (a3) Virtual-pole extension dnext[j] = d[j+1], dnext[k-1] = d[k-1]+gamma+mu
 * (pkg/src/hsseig/secular.py:195-199).  Needed by every Cauchy entry.
 */
int hsseig_dnext(const double *d, const double *gamma, const double *mu, int64_t k,
                 double *dnext, void *stream);

/*
 * (a4) Loewner recomputation of the weights.
 * Replaces recompute_weights (pkg/src/hsseig/secular.py:206-236).
 * status[3] = first index with a non-positive / non-finite radicand.
 */
int hsseig_loewner(const double *d, const double *dnext, const double *gamma,
                   const double *mu, const double *z, int64_t k, double rho, double *zhat,
                   hsseig_status *status, void *stream);
/* Weights [ibeg, iend) only; zhat holds iend - ibeg entries. */
int hsseig_loewner_part(const double *d, const double *dnext, const double *gamma,
                        const double *mu, const double *z, int64_t k, double rho, int64_t ibeg,
                        int64_t iend, double *zhat, hsseig_status *status, void *stream);

/*
 * (a5) Column normalizers v_j = 1/||zhat ./ (d - lam_j)||.
 * Replaces column_normalizers (pkg/src/hsseig/secular.py:239-250).
 */
int hsseig_normalizers(const double *d, const double *dnext, const double *gamma,
                       const double *mu, const double *zhat, int64_t k, double *v,
                       void *stream);
/* Normalizers of columns [jbeg, jend) only; v holds jend - jbeg entries. */
int hsseig_normalizers_part(const double *d, const double *dnext, const double *gamma,
                            const double *mu, const double *zhat, int64_t k, int64_t jbeg,
                            int64_t jend, double *v, void *stream);

/* Generators of the Cauchy-like matrix (pkg/src/hsseig/cauchy.py:15-38); device pointers. */
typedef struct hsseig_gen {
  const double *d, *dnext, *gamma, *mu, *zhat, *v;
  int64_t k;
} hsseig_gen;

/*
 * (a6) Dense block C[rows, cols] -> out (nr x nc, leading dim ldo).
 * Replaces CauchyEvecMatrix.block (pkg/src/hsseig/cauchy.py:48-56).
 * rows/cols: int64 device index arrays.
 */
int hsseig_cauchy_block(const hsseig_gen *gen, const int64_t *rows, int64_t nr,
                        const int64_t *cols, int64_t nc, double *out, int64_t ldo,
                        void *stream);

/*
 * (a7) Randomized sampling Y = C @ Omega and Z = C^T @ Omega with C generated
 * tile by tile in shared memory and contracted on FP64 DMMA.
 * Replaces CauchyEvecMatrix.multiply / transpose_multiply (cauchy.py:70-100).
 * Omega: k x w (ld = ldom, even; 16-byte aligned rows for TMA).  Y, Z: k x w (ld = ldy).
 * work: hsseig_sample_work_doubles(k, w) doubles (split-K partials).
 * leaf_of: NULL for the full products (the reference's C Omega, C^T Omega), or the tree's
 * leaf id per index (hsseig_tree.leaf_of) for the OFF-DIAGONAL sample the construction uses
 * by default: entries with leaf_of[i] == leaf_of[j] count as zero, so Y_t = Phi_t =
 * C(t, t^c) Omega(t^c) directly instead of Y_t - D_t Omega_t (hss.py:265-266), which cancels
 * the dominant diagonal block and leaves the sum's rounding noise for the ID to truncate
 * against (half the ranks, ~15x smaller HSS error at config 4's shape).
 */
int64_t hsseig_sample_work_doubles(int64_t k, int64_t w);
int hsseig_cauchy_sample(const hsseig_gen *gen, const int32_t *leaf_of, const double *omega,
                         int64_t ldom, int64_t w, double *Y, double *Z, int64_t ldy, double *work,
                         void *stream);
/* Rows [row0, row1) of Y and of Z (multi-GPU shard); Y, Z hold row1 - row0 rows. */
int hsseig_cauchy_sample_part(const hsseig_gen *gen, const int32_t *leaf_of, const double *omega,
                              int64_t ldom, int64_t w, int64_t row0, int64_t row1, double *Y,
                              double *Z, int64_t ldy, double *work, void *stream);

/*
 * Multi-GPU form fused with the all-gather: rows [row0, row1) of Y and Z are computed here
 * and stored by the split-K reduction kernels straight into every rank's full k x w Y / Z
 * (Yp / Zp: npeers device pointers, this rank's own included, IPC-mapped peer buffers over
 * NVLink / NVSwitch).  The caller synchronises its stream and barriers the group before
 * reading.  Materialised-panel path only (HSSEIG_ERR_ARG otherwise: use the NCCL gather).
 */
int hsseig_cauchy_sample_part_peers(const hsseig_gen *gen, const int32_t *leaf_of,
                                    const double *omega, int64_t ldom, int64_t w, int64_t row0,
                                    int64_t row1, const uint64_t *Yp, const uint64_t *Zp,
                                    int32_t npeers, int64_t ldy, double *work, void *stream);
/* 1 when hsseig_cauchy_sample_part_peers accepts a shard of `nrows` rows (order k, width w),
 * else 0.  Monotone in nrows: ranks evaluate it on the padded shard size they all share, so
 * every rank of a group takes the same path (peer stores or the NCCL gather). */
int hsseig_sample_peers_fits(int64_t k, int64_t nrows, int64_t w);

/*
 * HSS tree (pkg/src/hsseig/hss.py:151-214): nodes in the reference's postorder
 * numbering over a power-of-two leaf count.  Topology arrays are filled by the
 * host (hsseig_tree_layout); numeric slots by hsseig_hss_build_rand.
 * Slot layout (all row-major, leading dimension `ws`):
 *   U, V : n_nodes slots of pmax x ws; candidate row q at slot row q + 1 (row 0 is zero)
 *   Vt   : n_nodes slots of ws x pmax (V transposed; an inner node's right-child
 *          candidates start at the next even column)
 *   B    : n_nodes slots of ws x ws   (rU(node) x rV(sibling))
 *   D    : n_leaves slots of (dld + 2) x dld, D[a][b] at row a + 1 (dld = mmax rounded to even)
 *   ws   : w rounded up to a multiple of 16; every slot is zero outside its data
 *   rsel, csel, rloc, cloc : n_nodes x ws int32
 */
typedef struct hsseig_tree {
  int32_t k, n_leaves, depth, n_nodes, w, ws, pmax, mmax;
  /* device topology, indexed by postorder node id */
  const int32_t *lo, *hi, *left, *right;
  const int32_t *level_nodes; /* node ids ordered by (level, position), level 1..depth */
  const int32_t *level_off;   /* host-side copy is level_off_h */
  int32_t level_off_h[33];    /* offsets into level_nodes for levels 0..depth (+1) */
  int32_t root;
  /* device numeric slots */
  int32_t *rU, *rV, *rsel, *csel, *rloc, *cloc, *flags;
  double *U, *V, *Vt, *B, *D, *rres, *cres;
  int32_t dld;
  /* construction scratch (device) */
  double *M;      /* 2 * n_leaves * pmax * ws : matrices handed to the ID */
  double *psel;   /* n_nodes * ws * ws : selected rows of Phi */
  double *tsel;   /* n_nodes * ws * ws : selected rows of Theta */
  double *ycomp;  /* n_nodes * ws * ws : V^T Omega compressions */
  double *zcomp;  /* n_nodes * ws * ws : U^T Omega compressions */
  /* host-side upper bound on the node ranks, set by the caller after reading the ranks
     back (0 = unknown, w is used); sizes the multiply's output tiles to the ranks */
  int32_t rmax;
  /* device: leaf position of every index 0..k-1 (filled by hsseig_tree_layout); the
     leaf_of argument of the sampling calls for the off-diagonal sample */
  int32_t *leaf_of;
} hsseig_tree;

/*
 * (a10) Row interpolative decomposition M ~= X M[J, :] of a batch of p x w matrices
 * (pkg/src/hsseig/hss.py:104-148, interpolative_decomp / _interp_rows): column-pivoted
 * QR of M^T with dgeqp3 semantics, truncation where the trailing Frobenius mass of R
 * drops below (tol ||M||_F)^2 or at max_rank, saturation flag, X = identity on J.
 * Matrix b at M + b*stride_m (leading dimension ldm); X (p x max_rank, ldx) at
 * X + b*stride_x, J[b*max_rank ..], rank / resid / saturated per matrix.  Shared memory
 * per matrix: hsseig_interp_smem_bytes(p, w) <= 227 KB; w <= 128 (the sample widths).
 */
int64_t hsseig_interp_smem_bytes(int32_t p, int32_t w);
int hsseig_interp_decomp(const double *M, int64_t ldm, int64_t stride_m, int32_t p, int32_t w,
                         int64_t batch, double tol, int32_t max_rank, double *X, int64_t ldx,
                         int64_t stride_x, int32_t *J, int32_t *rank, double *resid,
                         int32_t *saturated, void *stream);

/* bytes of device memory hsseig_tree_layout carves for one tree */
int64_t hsseig_tree_bytes(int32_t k, int32_t n_leaves, int32_t w, int32_t mmax);
/*
 * Fill `tree` with pointers carved from `dev_mem` (hsseig_tree_bytes) and copy the
 * topology for leaf boundaries `bounds_h` (host, n_leaves+1 ints) to the device.
 */
int hsseig_tree_layout(hsseig_tree *tree, const int32_t *bounds_h, int32_t n_leaves, int32_t w,
                       void *dev_mem, void *stream);

/*
 * (a10, a11) Randomized HSS construction, Algorithm 2 (pkg/src/hsseig/hss.py:217-306):
 * leaf D / Phi / Theta formation, batched column-pivoted-QR interpolative
 * decompositions (dgeqp3 + dtrtrs semantics, hss.py:120-148) level by level,
 * skeleton B blocks regenerated from the generators.
 * Y, Z: sampled blocks (ld = ldy); omega (ld = ldom); w = r + p.  offdiag = 1: Y / Z are the
 * off-diagonal sample (hsseig_cauchy_sample with leaf_of), the leaves take Phi = Y_t,
 * Theta = Z_t; offdiag = 0: full products, Phi = Y_t - D Omega_t as hss.py:265-266.
 * status[4] = saturated-ID count (tree flagged), status[5] = r_used.
 */
int hsseig_hss_build_rand(const hsseig_gen *gen, const double *omega, int64_t ldom,
                          const double *Y, const double *Z, int64_t ldy, double id_tol,
                          int32_t offdiag, hsseig_tree *tree, hsseig_status *status,
                          void *stream);
/* Zero the tree's factor slots (done by hsseig_hss_build_rand; call once before the
 * per-level form below). */
int hsseig_tree_clear(hsseig_tree *tree, void *stream);
/*
 * Multi-GPU form: levels lev_from (deepest) .. lev_to only, and at every level only the
 * node positions of part `part` of `nparts` (power of two): each rank builds its own
 * subtrees below level log2(nparts); after the node slots are all-gathered the upper
 * levels are built (nparts = 1) on every rank.  lev_to = 0 also forms the root blocks.
 */
int hsseig_hss_build_rand_levels(const hsseig_gen *gen, const double *omega, int64_t ldom,
                                 const double *Y, const double *Z, int64_t ldy, double id_tol,
                                 int32_t offdiag, hsseig_tree *tree, hsseig_status *status,
                                 int lev_from, int lev_to, int part, int nparts, void *stream);

/*
 * (f4) ADC1: HSS construction by structured rank-revealing Schur complements (SRRSC) on the
 * generators, no sampling.  Named by BASELINE.json ("ADC1 (SRRSC HSS)") but absent from the
 * reference, so its definition is oracle/srrsc_oracle.py (parity unpinned).
 * Per node and side the block row C[R, t^c] (or column C[t^c, R]^T) is eliminated with
 * complete pivoting on its Cauchy-like generators until max|Schur| <= tol * max|block| or
 * max_rank steps (<= tree->w; saturation flag above 1e-12 as hss.py:117); the multipliers
 * give the interpolation bases, so U / V / B / D / skeletons fill the same slots as
 * hsseig_hss_build_rand and hsseig_hss_matmul_right applies the tree unchanged.
 * The replaced call site is the construction in update_vectors_hss (pkg/src/hsseig/dc.py:165).
 * work: hsseig_srrsc_work_doubles(tree) doubles (column generators per node and side).
 * status[4] = saturated count (tree flagged), status[5] = r_used.
 */
int64_t hsseig_srrsc_work_doubles(const hsseig_tree *tree);
int hsseig_hss_build_srrsc(const hsseig_gen *gen, double tol, int32_t max_rank, hsseig_tree *tree,
                           double *work, hsseig_status *status, void *stream);
/* Multi-GPU form (levels lev_from..lev_to, node positions of part `part` of `nparts`), with
 * the conventions of hsseig_hss_build_rand_levels. */
int hsseig_hss_build_srrsc_levels(const hsseig_gen *gen, double tol, int32_t max_rank,
                                  hsseig_tree *tree, double *work, hsseig_status *status,
                                  int lev_from, int lev_to, int part, int nparts, void *stream);

/*
 * (a12) Structured product out = X @ H (Algorithm 3; pkg/src/hsseig/hss.py:309-361).
 * X: P x k (ld = ldx), out: P x k (ld = ldo), row-major.
 * work: hsseig_matmul_work_doubles(P, tree) doubles.
 */
int64_t hsseig_matmul_work_doubles(int64_t P, const hsseig_tree *tree);
int hsseig_hss_matmul_right(const double *X, int64_t ldx, int64_t P, const hsseig_tree *tree,
                            double *out, int64_t ldo, double *work, void *stream);
/*
 * The same product in two parts: part 0 = the leaf up-level G = X U_leaf only (it reads
 * nothing above the tree's leaf level, so it may run on a second stream beside the
 * construction of the upper levels, on at most max_ctas SMs; 0 = no cap); part 1 = the
 * rest, once part 0 and the whole construction are done.  Same work buffer for both.
 */
int hsseig_hss_matmul_right_part(const double *X, int64_t ldx, int64_t P,
                                 const hsseig_tree *tree, double *out, int64_t ldo, double *work,
                                 int32_t part, int32_t max_ctas, void *stream);

/*
 * (a14) Dense update out = Qb @ C with C generated on the fly (fallback path).
 * Replaces update_vectors_dense(Qblock, C.to_dense()) (pkg/src/hsseig/dc.py:132-138).
 */
int hsseig_dense_update(const double *Qb, int64_t ldq, int64_t P, const hsseig_gen *gen,
                        double *out, int64_t ldo, void *stream);

/*
 * The reference's Gaussian sample draw on the device, bit-identical to
 * numpy.random.Generator(PCG64(state, inc)).standard_normal(n) (hss.py:236-237).
 * hsseig_set_normal_tables loads NumPy's ziggurat tables (ki, wi, fi; 256 each, host
 * pointers) once.  state/inc: the PCG64 128-bit state and increment as hi/lo words
 * (Generator.bit_generator.state).  Value i goes to out[(i / w) * ldo + i % w], i.e. the
 * row-major (n / w) x w block standard_normal((n / w, w)) with leading dimension ldo.
 * work: hsseig_normals_work_bytes(n) bytes.
 * *fail_dev (int32, device) is set non-zero if the rejection chain could not be
 * resolved; the caller then draws on the host instead.
 * tails (device int64, 1 + 3*tail_cap; may be NULL): tails[0] = count, then per normal
 * taken from the ziggurat tail (about 1 in 4000) its output offset, the raw 64-bit draw
 * fed to log1p and the sign bit.  NumPy evaluates those with the C library's log1p; the
 * host re-evaluates them (value = +-(r - log1p(-u) / r)) so the block is bit-identical.
 */
/*
 * Tail fix-up of a draw: h_tails is the host copy of the draw's tails block (pinned), the
 * values are re-evaluated with the C library's log1p (zig_r / zig_inv_r: NumPy's
 * ziggurat_nor_r and ziggurat_nor_inv_r) into h_pairs (pinned, 2*tail_cap int64) and
 * scattered into out on the stream by a kernel that reads them in place (mapped pinned
 * memory; d_pairs, device 2*tail_cap int64, is the staging used only where host memory
 * is not device-mapped).  Returns the
 * number of values fixed, or -status.  (The Python loop of the reference's own draw,
 * numpy/random/src/distributions/distributions.c random_standard_normal, tail branch.)
 */
int64_t hsseig_normals_fixup(const int64_t *h_tails, int64_t tail_cap, double zig_r,
                             double zig_inv_r, int64_t *h_pairs, int64_t *d_pairs, double *out,
                             void *stream);
int hsseig_set_normal_tables(const uint64_t *ki, const double *wi, const double *fi);
int64_t hsseig_normals_work_bytes(int64_t n);
int hsseig_pcg64_normals(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                         int64_t n, int64_t w, int64_t ldo, double *out, void *work,
                         int32_t *fail_dev, int64_t *tails, int64_t tail_cap, void *stream);

/* ---------------------------------------------------------------------------------------
 * Divide-and-conquer glue (the caller around the merge: SURVEY.md §8 f1-f2).
 * --------------------------------------------------------------------------------------- */
/*
 * Base case for every leaf of the recursion at once: implicit QL with Wilkinson shift
 * (tql2, pkg/src/hsseig/_kernels.pyx:352-411) followed by the ascending stable sort of
 * dc.py:118-129.  Matrix m has order off[m+1]-off[m] <= nmax <= 160 (a warp per matrix when
 * nmax <= 32, a 128-thread block per matrix above), diagonal a[off[m]..] and off-diagonal
 * b[off[m]-m..] (n-1 entries); lam[off[m]..] receives its eigenvalues and Q[qoff[m]..] its
 * n x n row-major eigenvectors.  status[m] = 1 + l if eigenvalue l stalls after max_iter
 * sweeps (BaseCaseError), else untouched.  flags bit 0: Q holds the initial accumulator Z
 * (in/out, the kernel contract tql2(d, e, Z)); bit 1: leave lam / Q in QL order (no sort).
 * nmax above 160 (the reference accepts any base_size >= 3) is HSSEIG_ERR_ARG.
 */
int hsseig_tql2_batched(const double *a, const double *b, const int64_t *off, int64_t nmat,
                        int nmax, int max_iter, double *lam, double *Q, const int64_t *qoff,
                        int32_t *status, int flags, void *stream);
/*
 * Host deflation of the merged system (pkg/src/hsseig/secular.py:91-156): returns k;
 * d_out/z_out/perm hold the kept system then the deflated poles; rotations (ri, rj, rc,
 * rs) in input indices, n_rot of them.  Host pointers.
 */
int64_t hsseig_deflate(const double *d, const double *z, int64_t n, double rho, double *d_out,
                       double *z_out, int64_t *perm, int64_t *ri, int64_t *rj, double *rc,
                       double *rs, int64_t *n_rot, double *tol_out);
/* The same with an explicit tolerance (deflate(..., eps_scale), secular.py:91-96). */
int64_t hsseig_deflate_tol(const double *d, const double *z, int64_t n, double rho, double tol,
                           double *d_out, double *z_out, int64_t *perm, int64_t *ri, int64_t *rj,
                           double *rc, double *rs, int64_t *n_rot);
/* W[:, c] = blockdiag(Q1, Q2)[:, src[c]] (dc.py:222-224, 241, 255). */
int hsseig_assemble_merge(const double *Q1, int64_t n1, const double *Q2, int64_t n2,
                          const int64_t *src, double *W, int64_t ldw, void *stream);
/* Deflation rotations on column pairs of W, in order (dc.py:225-230). */
int hsseig_apply_rotations(double *W, int64_t ldw, int64_t rows, const int64_t *ca,
                           const int64_t *cb, const double *c, const double *s, int64_t nrot,
                           void *stream);
/* out[:, c] = src[c] < k ? A[:, src[c]] : B[:, src[c]] (final eigenvalue order, dc.py:253-257). */
int hsseig_gather_columns(const double *A, int64_t lda, const double *B, int64_t ldb, int64_t k,
                          const int64_t *src, int64_t ncol, int64_t rows, double *out,
                          int64_t ldo, void *stream);

/* Multi-GPU merges (row-block sharded Q): one rank's rows, all from child c whose columns
   start at coff: W[i][c'] = Qc[i][src[c'] - coff] for src in [coff, coff + nc), else 0. */
int hsseig_assemble_rows(const double *Qc, int64_t ldq, int64_t nrow, int64_t coff, int64_t nc,
                         const int64_t *src, int64_t n, double *W, int64_t ldw, void *stream);

/* ---------------------------------------------------------------------------------------
 * Level-batched merges: every merge of one recursion depth of
 * adc_solve (pkg/src/hsseig/dc.py:194-257) in one set of launches.  Merge m has n1[m] +
 * n2[m] rows, concatenated at roff[m] (row_merge[r] = merge of row r); its children blocks
 * are at device addresses q1[m], q2[m] (row-major n1 x n1, n2 x n2); its n x n block
 * W_m at W + woff[m] with an even leading dimension n + (n & 1).  Kept rank-one systems s own roots [koff[s], koff[s+1]) of the
 * concatenated root arrays; seg_of[i] = system of root i.  st[s] as hsseig_status_init.
 * --------------------------------------------------------------------------------------- */
/* z rows: [last row of Q1, first row of Q2] per merge (dc.py:112). */
int hsseig_wave_zrows(const uint64_t *q1, const uint64_t *q2, const int64_t *n1,
                      const int64_t *n2, const int64_t *roff, int64_t nm, double *zrow,
                      void *stream);
/* Host: joint sort + deflation of every merge (dc.py:205-235, secular.py:91-156); src /
   d_out / z_out per row, rotations as W-column pairs [rot_off[m], rot_off[m+1]).  Returns
   the total kept roots. */
int64_t hsseig_wave_deflate(int64_t nm, const int64_t *n1, const int64_t *n2, const int64_t *roff,
                            const double *L, const double *zrow, const double *bk, int64_t *kept,
                            double *rho_eff, double *d_out, double *z_out, int64_t *src,
                            int64_t *rot_off, int64_t *ca, int64_t *cb, double *rc, double *rs);
/* Host: compact W layout (kept positions + deflated positions a rotation touches): widths
   wd, compact blockdiag columns csrc (offsets coff), position -> compact map cmap (-1: not
   materialised), rotation pairs rewritten to compact indices.  Returns the total width. */
int64_t hsseig_wave_compact(int64_t nm, const int64_t *roff, const int64_t *kept,
                            const int64_t *src, const int64_t *rot_off, int64_t *ca, int64_t *cb,
                            int64_t *wd, int64_t *coff, int64_t *csrc, int64_t *cmap);
/* Compact W_m (n x wd[m], leading dimension wd + (wd & 1)):
   W_m[:, j] = blockdiag(Q1, Q2)[:, csrc[coff[m] + j]]. */
int hsseig_wave_assemble(const uint64_t *q1, const uint64_t *q2, const int64_t *n1,
                         const int64_t *n2, const int64_t *roff, const int32_t *row_merge,
                         const int64_t *csrc, const int64_t *coff, const int64_t *wd, double *W,
                         const int64_t *woff, int64_t nrows, void *stream);
/* Deflation rotations of every merge on its W_m (dc.py:225-230).  A merge's rotations
 * (deflation's (survivor, deflated) pairs) split into runs sharing one survivor; run_t lists
 * the first rotation of every run over all merges plus a final sentinel (the rotation
 * count), run_off (nm + 1) each merge's first run.  Runs touch disjoint columns, so each
 * (row, run) pair is an independent task; max_tasks = max over merges of n_m * runs_m. */
int hsseig_wave_rotate(double *W, const int64_t *woff, const int64_t *n, const int64_t *wd,
                       const int64_t *run_t, const int64_t *run_off, const int64_t *ca,
                       const int64_t *cb, const double *c, const double *s, int64_t nm,
                       int64_t max_tasks, void *stream);
/* Secular roots of every kept system (secular_all per system); work: ntot + nseg doubles. */
int hsseig_wave_secular(const double *d, const double *z, const int64_t *koff,
                        const int32_t *seg_of, const double *rho, int64_t nseg, int64_t ntot,
                        double *lam, double *gamma, double *mu, int32_t *iters, double *work,
                        hsseig_status *st, void *stream);
int hsseig_wave_dnext(const double *d, const double *gamma, const double *mu, const int64_t *koff,
                      const int32_t *seg_of, int64_t ntot, double *dnext, void *stream);
int hsseig_wave_loewner(const double *d, const double *dnext, const double *gamma,
                        const double *mu, const double *z, const int64_t *koff,
                        const int32_t *seg_of, const double *rho, int64_t ntot, double *zhat,
                        hsseig_status *st, void *stream);
int hsseig_wave_normalizers(const double *d, const double *dnext, const double *gamma,
                            const double *mu, const double *zhat, const int64_t *koff,
                            const int32_t *seg_of, int64_t ntot, double *v, void *stream);
/* Grouped dense updates out_s = W_s[:, :k_s] @ C_s (dc.py:132-138); tasks: (s, row tile,
   column tile) int32 triples for tiles of hsseig_wave_tile_shape. */
int hsseig_wave_dense_update(const double *W, const int64_t *woff, const int64_t *nrow,
                             const int64_t *ldw, const double *d, const double *dnext, const double *gamma,
                             const double *mu, const double *zhat, const double *v,
                             const int64_t *koff, double *out, const int64_t *ooff,
                             const int32_t *tasks, int64_t ntasks, void *stream);
int hsseig_wave_tile_shape(int32_t *bm, int32_t *bn);
/* Host: final order of every merge: stable argsort of [roots, deflated poles]
   (dc.py:253-257). */
int hsseig_wave_order(int64_t nm, const int64_t *roff, const int64_t *kept, const int64_t *koff,
                      const double *lam, const double *d_out, int64_t *order, double *lam_out);
/* Column descriptors of the gather from the final order (local positions), the compact-W
   map (cmap, -1 = not materialised) and the blockdiag source columns (src). */
int hsseig_wave_desc(int64_t nm, const int64_t *roff, const int64_t *kept, const int64_t *order,
                     const int64_t *cmap, const int64_t *src, int64_t *desc);
/* out_m[:, c] from desc[roff[m] + c] = (source << 40) | index: source 0 = column of Qk_m
   (n x k_m), 1 = compact W_m column, 2 = blockdiag(Q1, Q2) column read from the children. */
int hsseig_wave_gather(const double *Qk, const int64_t *qoff, const int64_t *kept,
                       const double *W, const int64_t *woff, const int64_t *wd,
                       const int64_t *desc, const uint64_t *q1, const uint64_t *q2,
                       const int64_t *n1, const int64_t *n2, const int64_t *roff,
                       const int32_t *row_merge, double *out, const int64_t *ooff, int64_t nrows,
                       void *stream);
/* Rows sel_row[i] of merge sel_merge[i] of the same gather, written to out + sel_off[i]
 * (the boundary rows the next depth's z needs, dc.py:112, taken before the full gather). */
int hsseig_wave_gather_rows(const double *Qk, const int64_t *qoff, const int64_t *kept,
                            const double *W, const int64_t *woff, const int64_t *wd,
                            const int64_t *desc, const uint64_t *q1, const uint64_t *q2,
                            const int64_t *n1, const int64_t *n2, const int64_t *roff,
                            const int32_t *sel_merge, const int64_t *sel_row,
                            const int64_t *sel_off, int64_t nsel, double *out, void *stream);

/* The dense update through materialised column panels of C (the reference's to_dense
   entries) and the TMA/DMMA GEMM engine (k >= 512, 16-byte aligned Qb rows, even ldq);
   otherwise the same as hsseig_dense_update.  work: hsseig_dense_update_work_doubles(k,
   panel_cols) doubles for panels of up to panel_cols columns. */
int64_t hsseig_dense_update_work_doubles(int64_t k, int64_t panel_cols);
int hsseig_dense_update_ws(const double *Qb, int64_t ldq, int64_t P, const hsseig_gen *gen,
                           double *out, int64_t ldo, double *work, int64_t work_doubles,
                           void *stream);

/* The dense update of a DC merge (dc.py:132-138 applied to dc.py:215-235's block) without the
   structural zeros of blockdiag(Q1, Q2): perm (device, k entries) orders the kept columns as
   [child 1 only | touched by a deflation rotation | child 2 only]; rows [0, n1) of Qb
   contract over perm[0, ka) and rows [n1, P) over perm[kb, k) -- the terms the full product
   multiplies by exact zeros are skipped (LAPACK dlaed3's partition), about half the flops.
   work: hsseig_dense_update_halves_work_doubles(P, k, panel_cols) doubles, 16-byte aligned. */
int64_t hsseig_dense_update_halves_work_doubles(int64_t P, int64_t k, int64_t panel_cols);
int hsseig_dense_update_halves(const double *Qb, int64_t ldq, int64_t P, int64_t n1,
                               const hsseig_gen *gen, const int64_t *perm, int64_t ka,
                               int64_t kb, double *out, int64_t ldo, double *work,
                               int64_t work_doubles, void *stream);

/* hsseig_dense_update_halves for every panel update of one recursion depth (the solver's
   level-batched schedule): rec (host) holds 9 int64 per merge -- W offset, ldw, rows, n1,
   generator offset, k, ka, kb, out offset (offsets in doubles from W / the generator
   arrays / out); perm (device) holds the merges' K orders back to back.  The updates are
   dealt to up to nstreams (<= 8) internal side streams forked from and joined into `stream`,
   each with work_doubles / nstreams doubles of the workspace (each slice at least
   hsseig_dense_update_halves_work_doubles of the largest merge). */
int hsseig_wave_dense_halves(int64_t nbig, const int64_t *rec, const double *W, const double *d,
                             const double *dnext, const double *gamma, const double *mu,
                             const double *zhat, const double *v, const int64_t *perm,
                             double *out, double *work, int64_t work_doubles, int32_t nstreams,
                             void *stream);

/* Plain batched helper used by tests/bench: out = A @ B (P x K)(K x N), FP64 DMMA. */
int hsseig_gemm(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                int64_t ldc, int64_t M, int64_t N, int64_t K, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HSSEIG_B200_H */
