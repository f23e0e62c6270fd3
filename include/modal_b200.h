/*
 * modal_b200.h — C ABI of the B200-native Modal Γ projection library.
 *
 * The reference (`cmbproj`, pure Python/NumPy) has no FFI: its "plugin boundary" is the
 * Python call `gamma3d_matrix(tables, mapping, grid, ...)` (engine3d.py:156-186), reached by
 * module-level name binding (harness.py:21).  This header is the native boundary underneath
 * the drop-in Python mirror (`paper_1503_08809_b200.gamma3d_matrix`); every entry point names
 * the reference interface it replaces.  A ctypes binding of the kind a reference maintainer
 * would add is shown in INTEGRATION.md.
 *
 * Conventions
 *   - All array arguments are caller-owned, C-contiguous, row-major HOST pointers unless the
 *     name ends in `_dev` (then they are device pointers on `device`).
 *   - Multipoles are indexed l - l_min, exactly like BasisTables (basis.py:219-246).
 *   - Return codes: MG_OK=0; MG_EINVAL=1 (-> ValueError); MG_ENOMEM=2 (-> MemoryError);
 *     MG_ECUDA=3 (-> RuntimeError, CLI exit code 3 per cli.py:142-145).  The message of the
 *     last failure on the calling thread is returned by mg_last_error().
 *   - Calls are synchronous and blocking (like the reference).  Calls from several host
 *     threads are safe: executes on one device are serialised inside the library.
 *   - There is no CPU fallback: without a usable sm_100 device every compute entry point
 *     returns MG_ECUDA.
 */
#ifndef MODAL_B200_H
#define MODAL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MG_OK 0
#define MG_EINVAL 1
#define MG_ENOMEM 2
#define MG_ECUDA 3

#define MG_H2_GOSPER 0 /* h2_gosper, geometry.py:89-111 (bit-exact weights) */
#define MG_H2_EXACT 1  /* h2_exact via log-factorials, geometry.py:56-86 (few-ulp) */

/* Library version (major*10000 + minor*100 + patch). */
int mg_version(void);

/* Message of the last failed call on this thread ("" if none). */
const char* mg_last_error(void);

/* Number of visible CUDA devices (0 without a GPU; never fails). */
int mg_device_count(void);

/* Bounds-check counters of a CHECKED build (compiled with -DMG_CHECKED=1; compute-sanitizer is
 * not available on this pool): counts[i] = number of out-of-extent global writes / bulk-copy
 * source ranges seen at check site i (n <= 16 sites, see MgCheck in mg_gamma.cu) on `device`
 * since the last reset; *checked = 1 for a checked build, 0 otherwise (counts all zero). */
int mg_debug_checks(uint32_t* counts, int n, int reset, int* checked, int device);

/* ---------------------------------------------------------------------------------------
 * Domain: replaces TriangularDomain / enumerate_domain (geometry.py:145-200).
 * Ordered triples l1<=l2<=l3<=l_max, l3<=l1+l2, l1+l2+l3 even, lexicographic order
 * (geometry.py:161-171).  Requires 2 <= l_min <= l_max (geometry.py:154-155).
 * ------------------------------------------------------------------------------------- */

/* Total triple count and number of non-empty (l1,l2) rows of the reference enumeration.
 * Host-only arithmetic (no device needed). */
int mg_domain_count(int l_min, int l_max, int64_t* count, int64_t* rows);

/* Flat indices [begin,end) -> (l1,l2,l3), computed on the device from (l1,l2)-row prefix
 * sums (the domain is never materialised in full).  Bit-identical to domain.l1/l2/l3. */
int mg_domain_triples(int l_min, int l_max, int64_t begin, int64_t end, int32_t* l1,
                      int32_t* l2, int32_t* l3, int device);

/* If (l1,l2,l3)[count] is exactly the flat range [b, b+count) of the reference enumeration,
 * *begin = b; otherwise *begin = -1 (range detection for a user-built `domain` object,
 * engine3d.py:170-171: a contiguous slice runs through mg_gamma_sep, anything else through
 * mg_gamma_sep_triples).  One O(count) walk on the host, no device needed. */
int mg_domain_match_range(int l_min, int l_max, const int32_t* l1, const int32_t* l2,
                          const int32_t* l3, int64_t count, int64_t* begin);

/* zm[t] = _triple_z(...) * permutation_multiplicity(...) for flat t in [begin,end)
 * (engine3d.py:41-53,133-134; geometry.py:114-142), computed on the device.
 * h2_mode = MG_H2_GOSPER is bit-identical to NumPy; MG_H2_EXACT agrees to a few ulp.
 * C, v: [L] with L = l_max-l_min+1; C must be > 0 (ValueError otherwise, geometry.py:135). */
int mg_weights(int l_min, int l_max, const double* C, const double* v, int h2_mode,
               int64_t begin, int64_t end, double* zm, int device);

/* ---------------------------------------------------------------------------------------
 * Separable Γ: replaces gamma3d_matrix (engine3d.py:156-186) = make_plan + _sweep_chunk
 * (engine3d.py:123-136) + _block_accumulate (engine3d.py:86-120) + merge_partials
 * (scheduler.py:48-66).
 *   q     [p][L]       late-time basis      (BasisTables.q,        basis.py:228)
 *   qt    [p][Nx][L]   projected basis      (BasisTables.q_tilde,  basis.py:229)
 *   C, v  [L]                              (basis.py:230-231)
 *   wr2   [Nx]         integration_weights(r, integrator) * r**2 (engine3d.py:126)
 *   modes [n][3]       mapping.entries, i<=j<=k<p (basis.py:57-75)
 *   [begin,end)        flat range of the reference enumeration (a _sweep_chunk range);
 *                      begin=0,end=-1 means the whole domain.
 *   ndev, devs         the devices to shard over (devs NULL: 0..ndev-1; entries may repeat).
 *                      Like the reference's `workers` fork pool (engine3d.py:175-186) the
 *                      range is cut into ndev contiguous l2 slabs of equal modelled cost
 *                      (the full domain: exactly the mg_slab_plan bounds), each computed on
 *                      its device by its own host thread, and the partial Γ's are summed in
 *                      slab order (merge_partials) — bitwise reproducible for a device list.
 *   gamma [n][n]       output, overwritten; rows = late modes n, cols = primordial n'
 *                      (gamma.py:14-16).
 * ------------------------------------------------------------------------------------- */
int mg_gamma_sep(const double* q, const double* qt, const double* C, const double* v,
                 const double* wr2, const int64_t* modes, int p, int Nx, int n, int l_min,
                 int l_max, int h2_mode, int64_t begin, int64_t end, int ndev, const int* devs,
                 double* gamma);

/* Same, restricted to the (l2,l3)-rows whose l2 lies in [l2_begin,l2_end): the l2-slab
 * shard used by the multi-GPU path (one rank = one slab; partial Γ's add up exactly). */
int mg_gamma_sep_slab(const double* q, const double* qt, const double* C, const double* v,
                      const double* wr2, const int64_t* modes, int p, int Nx, int n,
                      int l_min, int l_max, int h2_mode, int l2_begin, int l2_end,
                      int device, double* gamma);

/* Same for an arbitrary explicit list of ordered valid triples (a user-built `domain`
 * object that is not a contiguous range, engine3d.py:170-171); sharded over ndev devices by
 * l2 slabs of the list like mg_gamma_sep. */
int mg_gamma_sep_triples(const double* q, const double* qt, const double* C,
                         const double* v, const double* wr2, const int64_t* modes, int p,
                         int Nx, int n, int l_min, int l_max, int h2_mode,
                         const int32_t* l1, const int32_t* l2, const int32_t* l3,
                         int64_t count, int ndev, const int* devs, double* gamma);

/* Balanced l2-slab boundaries for `nshards` ranks (cost model of the row-factorised kernel):
 * bounds[0..nshards] with bounds[0]=l_min, bounds[nshards]=l_max+1.  Host-only. */
int mg_slab_plan(int l_min, int l_max, int p, int Nx, int nshards, int* bounds);

/* ---------------------------------------------------------------------------------------
 * Resident plan (the bench's device-resident measurement and the multi-GPU ranks):
 * upload the tables once, then execute any number of Γ's / shards on device memory.
 * ------------------------------------------------------------------------------------- */
typedef struct mg_plan mg_plan;

int mg_plan_create(const double* q, const double* qt, const double* C, const double* v,
                   const double* wr2, const int64_t* modes, int p, int Nx, int n, int l_min,
                   int l_max, int h2_mode, int device, mg_plan** plan);
/* Same, but q̃ is taken from device memory laid out [p][Nx][L] (e.g. from mg_build_qtilde). */
int mg_plan_create_dev(const double* q, const double* qt_dev, const double* C,
                       const double* v, const double* wr2, const int64_t* modes, int p,
                       int Nx, int n, int l_min, int l_max, int h2_mode, int device,
                       mg_plan** plan);
/* Run the l2-slab [l2_begin,l2_end) (l2_end<0: to l_max) and leave Γ[n][n] in device
 * memory (gamma_dev, may be NULL: then only the plan's internal buffer is written).
 * stream: a cudaStream_t (NULL = legacy default stream).  Asynchronous w.r.t. the host. */
int mg_plan_execute(mg_plan* plan, int l2_begin, int l2_end, double* gamma_dev, void* stream);
/* Copy the plan's last Γ to host memory (synchronises the stream). */
int mg_plan_fetch(mg_plan* plan, double* gamma, void* stream);
/* Executed FP64 FLOPs of the last mg_plan_execute (per kernel family) and launch count. */
int mg_plan_stats(mg_plan* plan, double* flops_rowcontract, double* flops_xcontract,
                  double* flops_pairs, int64_t* launches);
/* Per-kernel-family timing with CUDA events on the launching stream (bench roofline):
 * after mg_plan_set_profile(plan, 1), every execute accumulates milliseconds into
 * ms[8] = {exposed wait of the contractions for their operands, run contraction,
 *          x contraction, R gather, pair contraction, final,
 *          operand kernels (A panels, pair products) on the side stream, overlapped,
 *          non-separable kernels (mg_plan_nonsep)}. */
int mg_plan_set_profile(mg_plan* plan, int on);
int mg_plan_kernel_ms(mg_plan* plan, double* ms);
void mg_plan_destroy(mg_plan* plan);

/* ---------------------------------------------------------------------------------------
 * Stage 1 (absent from the reference; equation):
 *   Δ_l(k)  = j_l(x_delta k) exp(-(k/k_damp)^2) (1 + eps_amp eps[l][k])
 *   C[l]    = Σ_k wk Δ_l(k)^2 / k
 *   q̃[c][x][l] = Σ_k wk k^2 qk[c][k] Δ_l(k) j_l(k x)
 * with j_l the spherical Bessel function from an on-device recurrence (upward for l<=kx,
 * Miller downward with exact power-of-two rescaling above), l = l_min..l_max.
 *   k, wk [Nk]; x [Nx]; eps [L][Nk]; qk [p][Nk].
 * Outputs (host): C [L], qt [p][Nx][L] (any may be NULL); delta [L][Nk] optional.
 * ------------------------------------------------------------------------------------- */
int mg_build_qtilde(const double* k, const double* wk, int Nk, const double* x, int Nx,
                    const double* eps, const double* qk, int p, int l_min, int l_max,
                    double x_delta, double k_damp, double eps_amp, int device, double* C,
                    double* qt, double* delta);
/* Same with device outputs (qt_dev [p][Nx][L], C_dev [L]); for the resident plan. */
int mg_build_qtilde_dev(const double* k, const double* wk, int Nk, const double* x, int Nx,
                        const double* eps, const double* qk, int p, int l_min, int l_max,
                        double x_delta, double k_damp, double eps_amp, int device,
                        double* C_dev, double* qt_dev, void* stream);

/* Spherical Bessel j_l(z) for l = 0..l_max at each z[i] (out [nz][l_max+1]); test hook
 * for the on-device generator (oracle: scipy.special.spherical_jn). */
int mg_bessel_table(const double* z, int nz, int l_max, int device, double* out);

/* ---------------------------------------------------------------------------------------
 * Non-separable direct path (BASELINE config 3; no reference counterpart — nearest are
 * radial_integral_x / late_product_y / gamma3d_naive, engine3d.py:56-83,189-215):
 *   B(t,x) = Σ_n' alpha[n'] Σ_6perms q̃q̃q̃(x; l1,l2,l3)     (pointwise, not factored)
 *   b[m]   = Σ_t W[t] zm[t] P[m,t] Σ_x wr2[x] B(t,x)
 * over an explicit list of ordered valid triples (l1,l2,l3,W) on a sparse l-grid.
 *   alpha [n]; out b [n].
 * ------------------------------------------------------------------------------------- */
int mg_gamma_nonsep(const double* q, const double* qt, const double* C, const double* v,
                    const double* wr2, const int64_t* modes, int p, int Nx, int n, int l_min,
                    int l_max, int h2_mode, const double* alpha, const int32_t* l1,
                    const int32_t* l2, const int32_t* l3, const double* W, int64_t count,
                    int device, double* b);
/* Resident form of the same path (tables of an mg_plan, sparse domain uploaded once):
 * mg_plan_set_sparse_domain validates and uploads (l1,l2,l3,W)[count]; mg_plan_nonsep
 * evaluates b for one alpha [n] (host) on `stream` into b_dev (device, optional) and/or
 * b_host (host, optional; synchronises).  With profiling on, kernel time accumulates in
 * mg_plan_kernel_ms()[7]. */
int mg_plan_set_sparse_domain(mg_plan* plan, const int32_t* l1, const int32_t* l2,
                              const int32_t* l3, const double* W, int64_t count);
int mg_plan_nonsep(mg_plan* plan, const double* alpha, double* b_dev, double* b_host,
                   void* stream);

/* ---------------------------------------------------------------------------------------
 * μ-quadrature ("separable", Modal2D) engine: replaces build_ptable / gamma2d_matrix
 * (engine2d.py:62-95, 187-211).
 *   lw [L] = (2l+1)/(v_l sqrt C_l); legendre [L][nmu] = P_l(μ_m) for l = l_min..l_max
 *   ptable [p][p][Nx][nmu] = Σ_l lw_l q_a(l) q̃_b(x,l) P_l(μ_m) (ascending-l Kahan, the
 *   reference's operation order: bit-identical table)
 *   gamma [n][n] = Σ_x wr2_x Σ_m mu_w[m] perm3(P[rows(n),cols(n')](x,m)) / (48π)
 * mg_gamma2d takes either a precomputed ptable or (q, qt, lw, legendre) to build it.
 * ------------------------------------------------------------------------------------- */
int mg_ptable(const double* q, const double* qt, const double* lw, const double* legendre,
              int p, int Nx, int L, int nmu, int device, double* ptable);
int mg_gamma2d(const double* q, const double* qt, const double* lw, const double* legendre,
               const double* ptable, const double* mu_w, const double* wr2,
               const int64_t* modes, int p, int Nx, int L, int nmu, int n, int device,
               double* gamma);
/* Kernel times (ms, CUDA events on the launching stream) of the calling thread's last
 * mg_ptable / mg_gamma2d call: the P-table kernel and the cell-sum kernels.  A stage that did
 * not run in that call (precomputed ptable) reports 0.  Measurement hook for bench.py; the
 * reference times the same two stages with perf_counter (harness.py:369-384). */
int mg_gamma2d_timings(double* ptable_ms, double* cells_ms);

#ifdef __cplusplus
}
#endif

#endif /* MODAL_B200_H */
