/*
 * domdec_b200.h — C ABI of the B200 domain-decomposition library.
 *
 * Every entry point takes plain device pointers (allocated by the host, e.g.
 * through torch), sizes and a cudaStream_t (passed as void*), enqueues its
 * kernels on that stream and returns 0 or a negative error code (the CUDA
 * error string is available from dd_last_error()).  No torch types cross
 * this boundary; the Python host layer (paper_2410_08859_b200/engine.py)
 * binds it with ctypes, exactly as a ctypes/cffi binding of the reference
 * package would.
 *
 * Problems are embedded as 2D grids: a 1D grid of n nodes is the 2D grid
 * (1, n).  A box is four int32 (off0, ext0, off1, ext1); an empty box has
 * ext0 == 0 or ext1 == 0.
 *
 * Reference interfaces replaced (paths under the reference package
 * pkg/src/domdec/):
 *   dd_grid_lse          sinkhorn.py:133-175   SeparableKernel.lse_x / lse_y
 *   dd_sinkhorn_run      sinkhorn.py:361-432   sinkhorn_solve (device-side iteration loop)
 *   dd_newton_global     sinkhorn.py:256-260   y_halfstep_newton, m = None branch
 *   dd_global_terms      sinkhorn.py:336-358   gap_kl_terms / _gap_kl
 *                        engine.py:654-662     StitchedGapEvaluator._dual_at sums
 *   dd_cell_solve        cells.py:165-393      make_cell_problems + solve_cell_batch
 *                                              (+ balance_cell_masses :446, _finalize :396)
 *   dd_cell_delta        engine.py:388-433     BlendScorer.__init__ (per-cell deltas)
 *   dd_blend_energy      engine.py:441-456     BlendScorer.energy_at
 *   dd_cell_commit       engine.py:726-785     _commit_cell + _stitch_alpha
 *   dd_assemble          measures.py:410-425   assemble_y_marginal (+ _masked: slab mode)
 *   dd_energy_terms      engine.py:185-196     PlanState.energy
 *   dd_product_init      engine.py:234-257     initial_plan_state (+ cells.py:566 product_plan_fragments)
 *   dd_cut_plan          engine.py:294-322     warm_start_plan (plan cut along basic cells)
 */
#ifndef DOMDEC_B200_H
#define DOMDEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Geometry and parameters of one transport problem (2D embedding). */
typedef struct dd_geom {
    int32_t nx0, nx1;          /* X grid dims */
    int32_t ny0, ny1;          /* Y grid dims */
    double x_dx, x_org0, x_org1;
    double y_dx, y_org0, y_org1;
    double eps, lam;
    double nu_total;           /* |nu| */
} dd_geom;

/* Device-resident plan state shared by the cell kernels. */
typedef struct dd_state {
    const double* mu;          /* X grid masses  [nx0*nx1] */
    const double* nu;          /* Y grid masses  [ny0*ny1] */
    const double* log_mu;      /* log mu (-inf where mu == 0) */
    const double* log_nu;
    int32_t n_basic;
    int32_t block0, block1;    /* basic block shape (s or 1, s) */
    const int32_t* basic_xbox; /* [n_basic*4] X block of each basic cell */
    const double* basic_mass;  /* [n_basic] mu mass per basic cell */
    int32_t* ybox;             /* [n_basic*4] Y-marginal boxes */
    double* yval;              /* [n_basic*cap] compact row-major values */
    int64_t cap;               /* slot capacity (entries) */
    double* x_marg;            /* [n_basic*block0*block1] dense over the block */
    double* transport;         /* [n_basic] */
    double* kl;                /* [n_basic] */
    /* dual store of the partition being processed */
    double* d_alpha;           /* [n_comp*nx_win] */
    int32_t* d_has;            /* [n_comp] */
    int32_t* d_box;            /* [n_comp*4] */
    double* d_beta;            /* [n_comp*d_cap] */
    int64_t d_cap;
} dd_state;

/* One batch of composite cells. Descriptor rows (int32, 12 per cell):
 *   j, xo0, xe0, xo1, xe1, yo0, ye0, yo1, ye1, n_mem, mem_base, flags
 * Offsets (int64, 4 per cell): y arena offset (ny entries), member arena
 * offset (6*n_mem*ny entries), workspace offset (global-memory mode),
 * member-x arena offset (n_mem*block entries). */
typedef struct dd_batch {
    int32_t n_cells;
    int32_t nxw0, nxw1;        /* common X window shape */
    const int32_t* desc;       /* [n_cells*12] */
    const int64_t* offs;       /* [n_cells*4] */
    const int32_t* members;    /* member basic ids */
    const double* snapshot;    /* assembled Y-marginal [ny0*ny1] */
    /* outputs / arenas */
    double* alpha;             /* [n_cells*nxw0*nxw1] */
    double* beta;              /* y arena: beta (in: warm start written by kernel) */
    double* mdens;             /* y arena: background density m */
    double* marena;            /* member arena */
    double* work;              /* workspace arena (global mode) */
    double* xarena;            /* member x-marginal arena */
    int32_t* mbox;             /* [n_members_total*4] new member boxes, by member slot */
    double* mstat;             /* [n_members_total*4] transport, kl, truncated, extra */
    double* cstat;             /* [n_cells*8] gap, first_gap, iters, conv, nclamped,
                                  newton_clamped, balance_fallbacks, target_miss */
    double* cstat2;            /* [n_cells*8] drift_nodes, trunc_total, loop cycles,
                                  Newton evaluations, executed Sinkhorn iterations
                                  (iters above is the reference-equivalent count),
                                  3 unused */
    int32_t smem_mode;         /* 1: workspace in shared memory */
    int32_t smem_bytes;
    /* solver configuration */
    double delta;              /* cell tolerance */
    int32_t max_iters;
    int32_t newton_max_iters;
    double newton_tol;
    double trunc;
    double* lnuw;              /* y arena: log nu on each cell window (kernel scratch) */
    double* lout;              /* [n_cells*nxw0*nxw1] final X sweep of cluster-solved cells */
    int32_t skip_stagnant;     /* 1: end a cell's loop early once an iteration reproduces
                                  beta bitwise (same results and reference iteration
                                  count; executed iterations in cstat2) */
    const int32_t* order;      /* nullable [n_cells]: CTA b of the solve kernel takes cell
                                  order[b] (longest-expected-first scheduling) */
    double* lmw;               /* y arena: log m on each cell window (kernel scratch) */
    int32_t split_smem_bytes;  /* > 0: cells flagged 4 run their Sinkhorn loop in a separate
                                  two-CTA-per-SM kernel with this much shared memory, then
                                  their epilogue in the solve kernel */
    int32_t precision;         /* 0: fp64; 1: fp32 mode (the single-CTA cell sweeps run
                                  in fp32: tables, weights, contractions; potentials,
                                  Newton, gap and epilogue fp64; north_star 1e-4) */
} dd_batch;

const char* dd_last_error(void);
int dd_device_count(void);
int dd_abi_version(void);

/* out = separable log-sum-exp sweep (to_x = 1: Y grid -> X grid). work holds
 * max(ny0*nx1, nx0*ny1) + max(nx0*ny0, nx1*ny1) doubles (intermediate + the
 * per-stage axis table). */
int dd_grid_lse(const dd_geom* g, const double* v, double* out, int to_x, double* work,
                void* stream);

/* Elementwise: out[i] = a[i]*s + b[i], or a[i]/s + b[i] when divide != 0
 * (b may be NULL). */
int dd_axpb(int64_t n, const double* a, double s, const double* b, double* out, int divide,
            void* stream);

/* Zero-background Y step: beta = finite(z) ? -ratio*z : lam*700; counts
 * degenerate nodes into *n_deg (device int, accumulated). */
int dd_newton_global(int64_t n, const double* z, double ratio, double lam, double* beta,
                     int32_t* n_deg, void* stream);

/* Per-node unbalanced Y step (sinkhorn.py:230-333): root of
 * log(m + exp(beta/eps + z)) + beta/lam = 0 by safeguarded Newton, with the
 * closed forms for m == 0 / z == -inf.  m == NULL means zero background;
 * eps and lam are per node. */
int dd_newton_nodes(int64_t n, const double* z, const double* m, const double* beta0,
                    const double* eps, const double* lam, double tol, int max_iters, double* beta,
                    int32_t* n_deg, void* stream);

/* Global reductions.  mode 0 (gap):  sums[0] = sum_x gap terms of
 *   KL(P_X pi | e^{-alpha/lam} mu) given L, px written if non-NULL.
 * mode 1 (dual): sums[0] = sum nu e^{b/eps + z}, sums[1] = sum mu(1-e^{-a/lam}),
 *   sums[2] = sum nu(1-e^{-b/lam}).  partial holds >= 2*1024 doubles. */
int dd_global_terms(int mode, int64_t n_x, int64_t n_y, const double* a, const double* l,
                    const double* w, const double* b, const double* z, const double* w2,
                    double eps, double lam, double* px, double* partial, double* sums,
                    void* stream);

/* Cell batch: assemble windows, Sinkhorn to tolerance, split, balance,
 * truncate, fragments, x-marginals. */
int dd_cell_solve(const dd_geom* g, const dd_state* s, const dd_batch* b, void* stream);

/* As dd_cell_solve, with the cells whose workspace does not fit shared memory
 * (n_big of them) handled on stream_big, concurrently with the shared-memory
 * cells on `stream` (joined back before return).  Of those, the cells listed
 * in clu_ids (device int32; their desc flags bit 0 set) run their Sinkhorn
 * loop on thread-block clusters, rows of the Y window split across the
 * cluster: host arrays goff[n_groups+1], gsize[n_groups], gsmem[n_groups]
 * give, per launch group, the slice of clu_ids, the cluster size (2..16) and
 * the shared memory per CTA.  Every big cell then goes through the
 * global-workspace kernel variant (max-L1 carveout), epilogue only for the
 * cluster-solved ones. */
int dd_cell_solve2(const dd_geom* g, const dd_state* s, const dd_batch* b, void* stream,
                   void* stream_big, int n_big, const int32_t* clu_ids, int n_groups,
                   const int32_t* goff, const int32_t* gsize, const int32_t* gsmem);

/* Minimum resident cell CTAs per SM the library was built for (1 or 2). */
int dd_cell_min_blocks(void);

/* Shared-memory doubles per CTA of the cluster variant. */
int64_t dd_cell_cluster_ws(int nw0, int nw1, int ny0, int ny1, int clu_size);

/* Blend scoring: per-cell dy windows (into dy arena at the y offsets) and
 * per-cell scalars cd[c*4] = t_delta, k_delta, d1_old, unused. */
int dd_cell_delta(const dd_geom* g, const dd_state* s, const dd_batch* b, double* dy,
                  double* cd, void* stream);

/* Tracked energy pieces for per-cell weights theta: ywork (grid) = snapshot
 * + sum theta dy, then out[0] = KL(clip(ywork) | nu), out[1..3] =
 * sum theta t_delta, sum theta k_delta, sum (d1_blend - d1_old). */
int dd_blend_energy(const dd_geom* g, const dd_state* s, const dd_batch* b, const double* dy,
                    const double* cd, const double* theta, double* ywork, double* partial,
                    double* out, void* stream);

/* Slab mode, rank-local parts of dd_blend_energy: dsum (Y grid) = sum_c theta_c dy_c
 * over the cells with theta_c != 0 (no snapshot base), out[1..3] = their summed
 * per-cell pieces, out[0] = 0.  The caller sums dsum and out over the ranks. */
int dd_blend_parts(const dd_geom* g, const dd_state* s, const dd_batch* b, const double* dy,
                   const double* cd, const double* theta, double* dsum, double* partial,
                   double* out, void* stream);

/* Commit theta-blends; stores duals, stitches alpha into alpha_grid, writes
 * per-cell errs[c*4] = x_err, y_err, truncated added, unused.  If yrun is
 * non-NULL it is updated in place (sequential mode). */
int dd_cell_commit(const dd_geom* g, const dd_state* s, const dd_batch* b, const double* theta,
                   double* alpha_grid, double* yrun, double* errs, void* stream);

/* out (Y grid) = sum of the basic-cell marginals, accumulated in cell index order
 * (fixed-order gather, bitwise reproducible). */
int dd_assemble(const dd_geom* g, const dd_state* s, double* out, void* stream);

/* Slab mode: the same sum over the basic cells whose mask entry is 1.0 (0.0 skips;
 * one double per basic cell). */
int dd_assemble_masked(const dd_geom* g, const dd_state* s, const double* mask, double* out,
                       void* stream);

/* sums[0] = sum transport, [1] = sum kl, [2] = sum_i KL(x_marg_i | mu_i),
 * [3] = KL(y | nu) for the given Y grid y. */
int dd_energy_terms(const dd_geom* g, const dd_state* s, const double* y, double* partial,
                    double* sums, void* stream);
/* Slab mode: sums[0..2] over the basic cells with mask 1.0 only; sums[3] as above. */
int dd_energy_terms_masked(const dd_geom* g, const dd_state* s, const double* y,
                           const double* mask, double* partial, double* sums, void* stream);

/* Product start nu_i = (m_i/|mu|) nu on the full box (cap >= ny0*ny1). */
int dd_product_init(const dd_geom* g, const dd_state* s, double mu_total, void* stream);

/* Cut the diagonal-scaling plan of global duals (alpha on X, beta on Y)
 * along the basic cells: fragments and x-marginals into the state, the
 * truncated bounding box of each cell's Y-marginal into boxes_out and the
 * removed mass into trunc_out[i].  Values are written into the slots when
 * s->yval is non-NULL and the box fits s->cap (call once with yval = NULL to
 * size the slots, then again to fill them).  Requires block0*block1 <= 64. */
int dd_cut_plan(const dd_geom* g, const dd_state* s, const double* alpha, const double* beta,
                double trunc, double* trunc_out, int32_t* boxes_out, void* stream);

/* Seed the dual store of one partition (n_comp cells, X windows xbox,
 * Y boxes ybox) from global duals. */
int dd_seed_duals(const dd_geom* g, const dd_state* s, int n_comp, int nw0, int nw1,
                  const int32_t* xbox, const int32_t* ybox, const double* alpha,
                  const double* beta, void* stream);

/* opt strategy (engine.py:465-503): lam-free derivative pieces of the blend
 * objective of cell c at weight th (th_cur = its current weight, ycur = the
 * running blended Y-marginal): out[0..3] = sum d log(x/mu), sum d^2/x,
 * sum dy log(y/nu), sum dy^2/y. */
int dd_opt_gh(const dd_geom* g, const dd_state* s, const dd_batch* b, const double* dy, int c,
              double th, double th_cur, const double* ycur, double* out, void* stream);

/* ycur on cell c's window = clip(ycur + dth * dy, 0). */
int dd_opt_set(const dd_geom* g, const dd_batch* b, const double* dy, int c, double dth,
               double* ycur, void* stream);

/* Multiscale refinement (SPEC multiscale.refine_plan): each fine basic cell
 * j takes its coarse parent's Y-marginal (parent[j]; coarse boxes/slots
 * cbox/cval with capacity ccap, coarse masses cmass, coarse nu grid nu_c of
 * row length cny1), split by fine mu mass and, within Y, by fine nu mass;
 * truncated at trunc (removed mass into trunc_out[j]); product-plan
 * fragments and x-marginals.  The fine slots must hold 4x the coarse box. */
int dd_refine(const dd_geom* g, const dd_state* s, const int32_t* parent, const int32_t* cbox,
              const double* cval, int64_t ccap, const double* cmass, const double* nu_c,
              int cny1, double trunc, double* trunc_out, void* stream);

/* Global unbalanced Sinkhorn iterations on the device (zero background):
 * iterations k0 .. k0+n_iters-1 of sinkhorn.py:361-432 are enqueued without host
 * synchronisation; the stopping test (gap/lam <= thr, checked at the top of every
 * iteration k >= 2) runs on the device and sets ctl_i[0]; ctl_i[1] = completed
 * iterations, ctl_d[0] = gap at the stop.  work holds dd_sinkhorn_ws(g) doubles
 * (axis tables built when tables_ready == 0, reused after).  L, px (X grid) and
 * z, bv, av (bv: Y grid, av: X grid) are scratch/outputs as in the host loop. */
int64_t dd_sinkhorn_ws(const dd_geom* g);
int dd_sinkhorn_run(const dd_geom* g, double* alpha, double* beta, const double* mu,
                    const double* log_mu, const double* log_nu, double* L, double* z, double* bv,
                    double* av, double* px, double* work, int* ctl_i, double* ctl_d, double thr,
                    int k0, int n_iters, int tables_ready, void* stream);

/* fp32-mode diagnostics: out[0..3] = fast-path X / Y sweeps redone by the fp64
 * stage-wise path, and all fp32 X / Y sweeps, since the last call (then reset). */
int dd_sweep_fallbacks(unsigned long long* out);

/* Bilinear prolongation of a cell-centred coarse field (nc0 x nc1) to the
 * x2 finer grid (nf0 x nf1); constant beyond the outer coarse centres. */
int dd_prolong(int nf0, int nf1, int nc0, int nc1, const double* coarse, double* fine,
               void* stream);

/* Workspace doubles one cell of the given window shape needs. */
int64_t dd_cell_ws_size(int nw0, int nw1, int ny0, int ny1);

/* out[q] = sum over rows of in[r*width + q] (fixed order), q < width. */
int dd_reduce_rows(int64_t n_rows, int width, const double* in, double* out, void* stream);

/* out[0] = sum KL(max(y,0) | nu) (clip != 0) or KL(y | nu). */
int dd_grid_kl(int64_t n, const double* y, const double* nu, int clip, double* partial,
               double* out, void* stream);

/* ==== three-axis (3D) path: csrc/vol.cu ====================================
 *
 * Problems of up to three axes embedded as 3D grids: a 2D grid (n0, n1) is
 * (1, n0, n1), a 1D grid (n) is (1, 1, n).  A box is six int32 (off0, ext0,
 * off1, ext1, off2, ext2); empty when any extent is 0.  The algorithm is the
 * reference's (same entry points as the 2D path above); the reference's own
 * Grid rejects 3D (measures.py:76-77) and its SeparableKernel reduces two
 * axes (sinkhorn.py:159-175) -- the three-axis sweep reduces axis 2, then 1,
 * then 0, the same order the 2D sweep uses for its two axes.
 *
 * Reference interfaces replaced (pkg/src/domdec/):
 *   dd3_grid_lse       sinkhorn.py:133-175   SeparableKernel.lse_x / lse_y (three axes)
 *   dd3_sinkhorn_run   sinkhorn.py:361-432   sinkhorn_solve (device-side iteration loop)
 *   dd3_prolong        SPEC multiscale       trilinear prolongation of duals
 *   dd3_cell_solve     cells.py:165-443      make_cell_problems + solve_cell_batch +
 *                                            balance_cell_masses + _finalize
 *   dd3_cell_delta     engine.py:388-433     BlendScorer.__init__ per-cell pieces
 *   dd3_cell_commit    engine.py:726-785     _commit_cell + _stitch_alpha
 *   dd3_gather         measures.py:410-425   assemble_y_marginal; BlendScorer.energy_at's
 *                                            y0 + sum theta dy (engine.py:441-456)
 *   dd3_cell_terms     engine.py:185-196     PlanState.energy per-cell pieces
 *   dd3_product_init   engine.py:234-257     initial_plan_state (+ cells.py:566)
 *   dd3_cut_plan       engine.py:294-322     warm_start_plan's plan cut
 *   dd3_seed_duals     engine.py:325-335     warm_start_plan's dual seeding
 */
typedef struct dd3_geom {
    int32_t nx[3];             /* X grid dims */
    int32_t ny[3];             /* Y grid dims */
    int32_t first_axis;        /* first real axis (0 for 3D, 1 for 2D, 2 for 1D) */
    int32_t pad_;
    double x_dx, y_dx;
    double x_org[3], y_org[3];
    double eps, lam;
    double nu_total;
} dd3_geom;

typedef struct dd3_state {
    const double* mu;          /* X grid masses */
    const double* nu;          /* Y grid masses */
    const double* log_mu;      /* log mu (-inf where mu == 0) */
    const double* log_nu;
    int32_t n_basic;
    int32_t block[3];          /* basic block shape */
    const int32_t* basic_xbox; /* [n_basic*6] */
    const double* basic_mass;  /* [n_basic] */
    int32_t* ybox;             /* [n_basic*6] Y-marginal boxes */
    double* yval;              /* [n_basic*cap] compact row-major values */
    int64_t cap;
    double* x_marg;            /* [n_basic*block volume] dense over the block */
    double* transport;         /* [n_basic] */
    double* kl;                /* [n_basic] */
    double* d_alpha;           /* dual store of the partition: [n_comp*nx_win] */
    int32_t* d_has;            /* [n_comp] */
    int32_t* d_box;            /* [n_comp*6] */
    double* d_beta;            /* [n_comp*d_cap] */
    int64_t d_cap;
} dd3_state;

/* One batch of composite cells.  desc (int32, 16 per cell):
 *   j, xbox[6], ybox[6], n_mem, mem_base, flags
 * offs (int64, 4 per cell): y arena offset (ny entries), member arena offset
 * (5*n_mem*ny entries: raw split / f, values, tc, tl, mc), workspace offset
 * (dd3_cell_ws_size doubles), member-x arena offset (n_mem*block entries). */
typedef struct dd3_batch {
    int32_t n_cells;
    int32_t nxw[3];            /* common X window shape */
    const int32_t* desc;
    const int64_t* offs;
    const int32_t* members;
    const double* snapshot;    /* assembled Y-marginal (Y grid) */
    double* alpha;             /* [n_cells*nx_win] */
    double* beta;              /* y arena */
    double* mdens;             /* y arena: background density m */
    double* work;              /* workspace arena */
    double* marena;            /* member arena */
    double* xarena;            /* member x-marginal arena */
    int32_t* mbox;             /* [n_members_total*6] new member boxes */
    double* mstat;             /* [n_members_total*4] transport, kl, truncated, unused */
    double* cstat;             /* [n_cells*8] gap, first_gap, iters, conv, nu_minus_clamped,
                                  newton_clamped, balance_fallbacks, target_miss */
    double* cstat2;            /* [n_cells*8] drift nodes, truncated total, executed
                                  iterations, sweep fallbacks, Newton evaluations, Sinkhorn
                                  loop cycles (clock64), 2 unused */
    double delta;
    int32_t max_iters;
    int32_t newton_max_iters;
    double newton_tol;
    double trunc;
    int32_t smem_doubles;      /* shared-memory doubles per cell CTA for the hot per-cell
                                  arrays (the host sizes it for the batch's largest window;
                                  a cell that does not fit keeps them in the workspace) */
    int32_t precision;         /* 0: fp64 sweeps; 1: fp32 mode (the six contractions, their
                                  tables and weights in fp32 with the linear part of the X-side
                                  potential absorbed into the tables; state, Newton, gap test
                                  and epilogue fp64; north_star tolerance 1e-4) */
} dd3_batch;

/* Workspace doubles of dd3_grid_lse for the geometry. */
int64_t dd3_grid_ws(const dd3_geom* g);
/* Separable three-axis log-sum-exp over the full grids (to_x = 1: Y grid -> X grid).
 * work holds dd3_grid_ws(g) doubles, including one set of per-axis kernel tables per
 * direction; tables_ready != 0 reuses the set a previous call with the same geometry,
 * eps and direction built. */
int dd3_grid_lse(const dd3_geom* g, const double* v, double* out, int to_x, double* work,
                 int tables_ready, void* stream);
/* Global unbalanced Sinkhorn on the device over three axes (dd_sinkhorn_run's contract):
 * iterations k0 .. k0+n_iters-1 enqueued without host synchronisation, stopping test on
 * the device (ctl_i[0] stopped, ctl_i[1] iterations, ctl_d[0] gap); work holds
 * dd3_sinkhorn_ws(g) doubles (grid-LSE tables built when tables_ready == 0). */
int64_t dd3_sinkhorn_ws(const dd3_geom* g);
int dd3_sinkhorn_run(const dd3_geom* g, double* alpha, double* beta, const double* mu,
                     const double* log_mu, const double* log_nu, double* L, double* z, double* bv,
                     double* av, double* px, double* work, int* ctl_i, double* ctl_d, double thr,
                     int k0, int n_iters, int tables_ready, void* stream);
/* Trilinear prolongation of a cell-centred coarse field to the x2 finer grid. */
int dd3_prolong(const int32_t* nf, const int32_t* nc, const double* coarse, double* fine,
                void* stream);
/* Workspace doubles one cell needs (X window w[3], Y window n[3]). */
int64_t dd3_cell_ws_size(const int32_t* w, const int32_t* n);
/* Cell batch: windows, Sinkhorn to tolerance, split, balance, truncate, fragments. */
int dd3_cell_solve(const dd3_geom* g, const dd3_state* s, const dd3_batch* b, void* stream);
/* Per-cell blend pieces: dy windows (y arena offsets) and cd[c*8] = t_delta, k_delta,
 * d1_old, d1 at theta = 1, d1 at theta = theta_safe, 3 unused. */
int dd3_cell_delta(const dd3_geom* g, const dd3_state* s, const dd3_batch* b, double theta_safe,
                   double* dy, double* cd, void* stream);
/* Commit theta-blends (per cell theta[c]); stores duals, stitches alpha into alpha_grid
 * (nullable); errs[c*4] = x_err, y_err, truncated mass added, unused.  If yrun is
 * non-NULL it is updated in place: += new window - old window, clipped at 0
 * (iteration_sequential, engine.py:829-830; one cell per call). */
int dd3_cell_commit(const dd3_geom* g, const dd3_state* s, const dd3_batch* b,
                    const double* theta, double* alpha_grid, double* yrun, double* errs,
                    void* stream);
/* opt strategy (engine.py:378-527): out[c] = lam * sum over cell c's members of
 * KL((1 - theta[c]) x_old + theta[c] x_new | mu) (BlendScorer._d1_blend). */
int dd3_blend_d1(const dd3_geom* g, const dd3_state* s, const dd3_batch* b,
                 const double* theta, double* out, void* stream);
/* Coordinate-descent pieces of cell c (_coordinate_root's g_and_h, lam-free):
 * out[0..1] = X-side sum d log(x/mu), sum d^2/x; out[2..3] = Y-side sum dy log(y/nu),
 * sum dy^2/y with y = clip(clip(ycur - th_cur dy, 0) + th dy, 0). */
int dd3_opt_gh(const dd3_geom* g, const dd3_state* s, const dd3_batch* b, const double* dy,
               int c, double th, double th_cur, const double* ycur, double* out, void* stream);
/* ycur[window of cell c] = clip(ycur + dth * dy_c, 0) (BlendScorer.set_theta). */
int dd3_opt_set(const dd3_geom* g, const dd3_batch* b, const double* dy, int c, double dth,
                double* ycur, void* stream);
/* out (Y grid) = base (nullable: 0) + sum_i scale_i * v_i over item boxes, accumulated in
 * item order (product rounded before the add).  Item i: box at box + i*bstride, values
 * at vals + (voff ? voff[i] : i*vstride), compact row-major over its box; scale nullable.
 * kl_mode 1/2: partial[k] gets per-CTA sums of KL(y | nu) terms (2: y clipped at 0
 * first), *n_partial their count. */
int dd3_gather(const dd3_geom* g, int n, const int32_t* box, int bstride, const double* vals,
               int64_t vstride, const int64_t* voff, const double* scale, const double* base,
               double* out, int kl_mode, const double* nu, double* partial, int* n_partial,
               void* stream);
/* Per basic cell: out[i*4] = transport_i, kl_i, KL(x_marg_i | mu_i), 0. */
int dd3_cell_terms(const dd3_geom* g, const dd3_state* s, double* out, void* stream);
/* Product start nu_i = (m_i/|mu|) nu on the full box (cap >= grid size). */
int dd3_product_init(const dd3_geom* g, const dd3_state* s, double mu_total, void* stream);
/* Plan cut of global duals along the basic cells (two calls: yval NULL sizes the boxes).
 * tile_max is the workspace: dd3_cut_tiles(g) doubles.
 * Terms whose log value is below cut_log (e.g. -60) are skipped; tiles of Y nodes are
 * culled by a bound on that value.  tile_max holds dd3_cut_tiles(g) doubles. */
int64_t dd3_cut_tiles(const dd3_geom* g);
int dd3_cut_plan(const dd3_geom* g, const dd3_state* s, const double* alpha, const double* beta,
                 double trunc, double cut_log, double* tile_max, double* trunc_out,
                 int32_t* boxes_out, void* stream);
/* Seed one partition's dual store from global duals (xbox/ybox: [n_comp*6]). */
int dd3_seed_duals(const dd3_geom* g, const dd3_state* s, int n_comp, const int32_t* nxw,
                   const int32_t* xbox, const int32_t* ybox, const double* alpha,
                   const double* beta, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DOMDEC_B200_H */
