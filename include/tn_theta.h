/*
 * tn_theta.h — C ABI of the B200 (sm_100a) charge-sectored two-site Θ(c) builder.
 *
 * What it computes (Supplementary Eq. S5 "\label{theta}"):
 *
 *   Θ(c)[α,β] = λl[α] λr[β] Σ_{α_k} Σ_{j_k,j_{k+1}} U^{i_k,i_{k+1}}_{j_k,j_{k+1}} Γk[α,α_k] λk[α_k] Γk1[α_k,β]
 *               × δ(c_l−c_c−j_k) δ(c_c−c_r−j_{k+1}) δ(c_l−c−i_k) δ(c−c_r−i_{k+1}),      0 ≤ c ≤ N
 *
 * with c_l, c_c, c_r the bond charges ("photons to the right") of α = α_{k−1},
 * α_k and β = α_{k+1}, 0 ≤ i, j ≤ d−1, and U the two-mode gate of Eq. S4
 * (PAPER.md:56-58). The δ's are enforced by charge-block indexing, never stored.
 *
 * Conventions shared by every call (DESIGN.md §2 "Readings"):
 *   - Complex numbers are interleaved (re, im) pairs of IEEE double (cuDoubleComplex layout);
 *     a "complex pointer" below is a `double*` to 2·count doubles.
 *   - Bonds are sorted by charge, ascending and stable. perm_x[p] is
 *     the caller's bond index at sorted position p; off_x[q] = #bonds of charge < q (q = 0..N+1).
 *   - Θ(c) is a compact row-major R_c×C_c matrix (ld = C_c). Its rows are the sorted left
 *     positions [off_l[c], off_l[min(N,c+d−1)+1]) and its columns the sorted right positions
 *     [off_r[max(0,c−d+1)], off_r[c+1]) (R2). With world_size > 1 a rank holds the
 *     "local slab": the rows of Θ(c) that fall in its shard [r0, r1) of sorted left positions.
 *   - U is "packed": blocks n = 0..min(N, 2d−2) of fixed total photon number n, block n at
 *     offset Σ_{m<n} s_m², s_n = min(n,d−1) − max(0,n−d+1) + 1, entry [i][j] at
 *     (i − lo_n)·s_n + (j − lo_n), lo_n = max(0, n−d+1), value ⟨i, n−i|U|j, n−j⟩ (R5/R6).
 *   - Device pointers are CUDA device (or managed) memory on the current device; "host" pointers
 *     are ordinary CPU memory. The library never frees caller memory.
 *   - No call aborts the process. Every call returns a tn_status; tn_last_error() gives a
 *     thread-local human-readable detail for the most recent failure.
 *   - There is no CPU fallback: every computing step runs in this library's sm_100a kernels.
 */
#ifndef TN_THETA_H
#define TN_THETA_H

#include <stdint.h>

#if defined(__GNUC__)
#define TN_API __attribute__((visibility("default")))
#else
#define TN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TN_OK = 0,
  TN_ERR_DOMAIN = 1,       /* argument outside its domain: d<2, N<0, N>TN_MAX_N, χ<1, charge ∉ [0,N], non-finite θ/φ, c ∉ [0,N] */
  TN_ERR_DIMENSION = 2,    /* NULL pointer for a non-empty buffer, bad bond id */
  TN_ERR_CONSISTENCY = 3,  /* plan / communicator mismatch (world size, rank), plan not sharded */
  TN_ERR_CUDA = 4,         /* a CUDA runtime error (launch / copy / sticky fault) */
  TN_ERR_OOM = 5,          /* device or host allocation failed */
  TN_ERR_NCCL = 6,         /* NCCL missing or an NCCL call failed */
  TN_ERR_UNSUPPORTED = 7   /* a size limit of this build was exceeded (e.g. min(N+1,d) > TN_MAX_MIX) */
} tn_status;

#define TN_MAX_N 100        /* largest photon number N (charges 0..N) this build accepts */
#define TN_MAX_MIX 64       /* largest U-mix vector length min(N+1, d) */

typedef struct tn_plan tn_plan;   /* opaque; owns device tables + staging workspace */
typedef struct tn_comm tn_comm;   /* opaque; wraps an NCCL communicator */
typedef void* tn_stream;          /* a cudaStream_t (0 = legacy default stream) */

enum { TN_BOND_LEFT = 0, TN_BOND_CENTER = 1, TN_BOND_RIGHT = 2 };
enum { TN_GATHER_NONE = 0, TN_GATHER_ROOT = 1, TN_GATHER_SECTOR_OWNER = 2 };
enum { TN_BCAST_NONE = 0, TN_BCAST_SLABS = 1, TN_BCAST_FULL = 2 };

/* One entry of a Θ gather schedule (tn_plan_gather_schedule / tn_gather_schedule_host): rank `src`'s slab
 * of sector `sector` — `rows` × `cols` complex, row-major — lands at row `row_begin` of the FULL Θ(sector)
 * on rank `dst`. Entries with src == dst are placed in place by the exec (no transfer). */
typedef struct {
  int64_t sector, src, dst, row_begin, rows, cols;
} tn_transfer;

/* ------------------------------------------------------------------------------------------ */
/* Plan: bond re-indexing (K1) + work decomposition. Not on the hot path; synchronises once.   */
/* ------------------------------------------------------------------------------------------ */
/* tn_theta_plan — PAPER.md:90-94 ("sort the bonds according to their charges").
 *   d        local Fock dimension (occupations 0..d−1), d ≥ 2.
 *   N        total photon number; charges lie in [0, N]; 0 ≤ N ≤ TN_MAX_N.
 *   chi_*    bond dimensions of α_{k−1} (l), α_k (c), α_{k+1} (r); each ≥ 1.
 *   q_*      int32 charge per bond index, in the caller's bond order; host OR device pointers
 *            (told apart with cudaPointerGetAttributes). Read during the call only. Device charges are
 *            read on the plan's own stream, unordered with the caller's streams: the caller makes them
 *            ready first (e.g. synchronises the producing stream; the Python binding does).
 *   world_size, rank   row sharding of Θ over ranks (1, 0 for a single GPU). The plan computes
 *            flop-balanced shards of the sorted left positions and keeps the work for `rank`.
 *   out      receives the new plan; free with tn_plan_destroy.
 * Runs the K1 counting-sort kernel on an internal stream, copies the offset tables back, builds the
 * c_c-group tile list and sector tables, allocates the staging workspace.
 * Errors: TN_ERR_DOMAIN (d<2, N<0 or > TN_MAX_N, χ<1, a charge ∉ [0,N], world_size<1,
 * rank ∉ [0,world_size)), TN_ERR_UNSUPPORTED (min(N+1,d) > TN_MAX_MIX), TN_ERR_DIMENSION (NULL q),
 * TN_ERR_OOM, TN_ERR_CUDA. On error *out is NULL. */
TN_API tn_status tn_theta_plan(int d, int N, int64_t chi_l, int64_t chi_c, int64_t chi_r,
                        const int32_t* q_l, const int32_t* q_c, const int32_t* q_r,
                        int world_size, int rank, tn_plan** out);

/* tn_theta2_plan — the MPO (vectorized density operator) variant, PAPER.md:101, :107 ("MPOs are
 * vectorized into the MPS form, U → U⊗U*, and two conserved charges are present"; SPEC.md:142-150,
 * :348-356). Every bond carries a charge PAIR (q1, q2) ∈ [0, N]² (ket and bra photon numbers to the
 * right); bonds are sorted by the lexicographic key q1·(N+1) + q2, stable. The plan's
 * sectors are Θ(c1, c2), indexed s = c1·(N+1) + c2 ∈ [0, (N+1)²) in every query and in theta_out;
 * Θ(c1,c2) is compact row-major, rows = sorted left positions with l1−c1, l2−c2 ∈ [0, d−1], columns
 * = sorted right positions with c1−r1, c2−r2 ∈ [0, d−1] (R16–R18). tn_build_bs_unitary and
 * tn_theta_exec are used unchanged (exec applies U to species 1 and conj(U) to species 2);
 * tn_plan_offsets returns (N+1)²+1 entries over the keys. world_size/rank shard the sorted left
 * positions flop-balanced as in tn_theta_plan; a rank's slab of Θ(c1,c2) is the contiguous run of its
 * rows inside [r0, r1) (tn_plan_local_sector_shape gives its first row). tn_theta_exec_sharded accepts
 * pair plans with every gather mode (sector owners by the same LPT rule over the (N+1)² sectors).
 * Errors: as tn_theta_plan, plus TN_ERR_UNSUPPORTED when (N+1)² exceeds this build's sector limit
 * (N ≤ 9). */
TN_API tn_status tn_theta2_plan(int d, int N, int64_t chi_l, int64_t chi_c, int64_t chi_r,
                                const int32_t* q1_l, const int32_t* q2_l, const int32_t* q1_c,
                                const int32_t* q2_c, const int32_t* q1_r, const int32_t* q2_r,
                                int world_size, int rank, tn_plan** out);

TN_API tn_status tn_plan_destroy(tn_plan* plan);  /* NULL is accepted. */

/* Full Θ(c) shape R_c × C_c (all ranks). c is a sector index: c ∈ [0, N], or s = c1·(N+1)+c2 ∈
 * [0, (N+1)²) for pair plans. TN_ERR_DOMAIN for an index outside that range. */
TN_API tn_status tn_plan_sector_shape(const tn_plan* plan, int c, int64_t* R, int64_t* C);
/* This rank's slab of Θ(c): *R local rows × *C, its first row being row *row_begin of Θ(c). */
TN_API tn_status tn_plan_local_sector_shape(const tn_plan* plan, int c, int64_t* R, int64_t* C,
                                     int64_t* row_begin);
/* Copy perm_x (χ_x int32) / off_x (N+2 int32; (N+1)²+1 over the pair keys for pair plans) of bond x
 * into caller HOST memory. */
TN_API tn_status tn_plan_perm(const tn_plan* plan, int bond, int32_t* host_out);
TN_API tn_status tn_plan_offsets(const tn_plan* plan, int bond, int32_t* host_out);
/* Sorted-left-position shard [r0, r1) of rank r (any r in [0, world_size)). */
TN_API tn_status tn_plan_shard_rows(const tn_plan* plan, int r, int64_t* r0, int64_t* r1);
/* Receiving rank of sector c under TN_GATHER_SECTOR_OWNER: longest-processing-time assignment of the
 * sectors by element count R_c·C_c (largest first onto the least-loaded rank; ties → lower rank). */
TN_API tn_status tn_plan_sector_owner(const tn_plan* plan, int c, int* owner);
/* Useful work, 8 flops per complex MAC; any output pointer may be NULL.
 *   f_contract = 8 Σ_{allowed (c_l,c_c,c_r)} n_l n_c n_r  (whole problem),
 *   f_mix      = 8 Σ_{(c_l,c_r)} n_l n_r #c #c_c           (whole problem; pair plans: 8 Σ n_l n_r
 *                (L1²L2 + L1L2²), the U⊗U* mix applied one species at a time, R19),
 *   f_exec     = complex flops this rank's K4 executes incl. tile padding (8 per CMAC; for the
 *                paper-literal engine its per-sector GEMMs),
 *   f_contract_local, f_mix_local = this rank's share (its rows [r0, r1)). */
TN_API tn_status tn_plan_flops(const tn_plan* plan, int64_t* f_contract, int64_t* f_mix, int64_t* f_exec,
                               int64_t* f_contract_local, int64_t* f_mix_local);
/* Number of complex entries of the packed U for this (d, N). */
TN_API tn_status tn_plan_u_size(const tn_plan* plan, int64_t* n_entries);
/* Device bytes the plan owns (tables + staging workspace). */
TN_API tn_status tn_plan_workspace_bytes(const tn_plan* plan, int64_t* bytes);

/* Per-kernel device times (CUDA events recorded on the launching streams) of the most recent
 * calls made with this plan: ms[0] K1 bond sort (inside tn_theta_plan), ms[1] K2 U build,
 * ms[2] K3 staging, ms[3] K4 contraction, ms[4] K5 U-mix (pair plans: both K5P passes; the fused
 * and paper-literal engines report their whole contraction as K4 and ~0 for K5). Waits for those
 * events. Entries for calls not yet made are −1. */
TN_API tn_status tn_plan_kernel_times(const tn_plan* plan, float* ms5);
/* Number of kernel launches one tn_theta_exec on this plan makes with its current contraction engine
 * (the sector-table update k_set_sectors, K3/K3O/K3L staging, K4/K4O/K4L, and one K5 launch per non-empty
 * register class of the mix — pair plans: per K5P pass, single- and multi-value tiles; the plan's K1 and
 * tn_build_bs_unitary's K2 are one launch each on top). HOST output. Errors: DIMENSION. */
TN_API tn_status tn_plan_exec_launches(const tn_plan* plan, int64_t* n_launches);

/* Contraction engine of tn_theta_exec (default TN_CONTRACT_F64_DMMA):
 *   TN_CONTRACT_F64_DMMA   — FP64 tensor cores (DMMA.8x8x4), complex products in the 3-multiplication
 *                            form; rounding error ~1e-16 relative.
 *   TN_CONTRACT_INT8_OZAKI — FP64-accurate emulation on the tcgen05 INT8 tensor cores: each real
 *                            operand is split into `slices` signed 7-bit slices with per-row (A) /
 *                            per-column (B) power-of-two scales; slice products accumulate exactly in
 *                            int32 TMEM per diagonal p+q ≤ slices+1 and are recombined in FP64.
 *                            Truncation error ≈ √K·2^(−7·slices) relative (slices = 7: ~1e-13).
 * slices ∈ [4, 8] (ignored for DMMA). Builds the slice layout (pooled workspace) and syncs once.
 * Errors: TN_ERR_DOMAIN (unknown mode / slices out of range), TN_ERR_OOM, TN_ERR_CUDA,
 * TN_ERR_UNSUPPORTED (the literal engine on a pair plan).
 *   TN_CONTRACT_PAPER_LITERAL — ABLATION only: the paper's kernel shape, one
 *                            GEMM per Θ(c) over all its centre segments with the U element looked up per
 *                            output element at every segment boundary, no product-once reformulation and
 *                            no K5 (≈12× the flops at config 3). Same DMMA mainloop; single-charge plans.
 */
enum { TN_CONTRACT_F64_DMMA = 0, TN_CONTRACT_INT8_OZAKI = 1, TN_CONTRACT_PAPER_LITERAL = 2 };
TN_API tn_status tn_plan_set_contraction(tn_plan* plan, int mode, int slices);
TN_API tn_status tn_plan_get_contraction(const tn_plan* plan, int* mode, int* slices);

/* ------------------------------------------------------------------------------------------ */
/* U builder (K2) — Eq. S4, "O(d^4) for initializing U".        */
/* ------------------------------------------------------------------------------------------ */
/* Writes the packed beam-splitter blocks exp[θ(e^{iφ} a†b − e^{−iφ} a b†)] (a = mode k,
 * DESIGN.md R5) into U_out: a DEVICE complex pointer of tn_plan_u_size entries, caller-owned.
 * Each element is the closed-form binomial sum evaluated in double-double, rounded once.
 * Stream-ordered, no host sync. Errors: TN_ERR_DOMAIN (θ or φ not finite),
 * TN_ERR_DIMENSION (U_out NULL), TN_ERR_CUDA. */
TN_API tn_status tn_build_bs_unitary(const tn_plan* plan, double theta, double phi, tn_stream stream,
                              double* U_out);

/* ------------------------------------------------------------------------------------------ */
/* Exec: K3 staging → K4 grouped complex DMMA contraction → K5 U-mix + outer-λ epilogue.       */
/* ------------------------------------------------------------------------------------------ */
/* tn_theta_exec — Eq. S5 for every sector c = 0..N.
 *   gamma_k   DEVICE complex [χ_l × χ_c] row-major, caller bond order (Γ^{[k]}).
 *   lambda_k  DEVICE double [χ_c] (λ^{[k]}).
 *   gamma_k1  DEVICE complex [χ_c × χ_r] row-major (Γ^{[k+1]}).
 *   lambda_l  DEVICE double [χ_l] (λ^{[k−1]}),  lambda_r DEVICE double [χ_r] (λ^{[k+1]}).
 *   U         DEVICE packed complex U (from tn_build_bs_unitary or any caller-built U of the
 *             same layout — the library cannot check which gate it is).
 *   theta_out HOST array of N+1 DEVICE complex pointers; theta_out[c] receives this rank's
 *             slab of Θ(c) (R×C from tn_plan_local_sector_shape), row-major, ld = C. Entries
 *             with R·C = 0 may be NULL. Buffers must not alias the inputs or each other.
 * Γ entries outside δ-allowed charge blocks are never read. Stream-ordered, no host sync.
 * The plan's workspace is reused: one exec per plan in flight at a time. Capturable into a CUDA graph
 * (independent launches fork onto per-thread auxiliary streams and join back): a captured call waits on the
 * host for the plan's table upload, and the plan must outlive every graph (and replay) that contains it —
 * tn_plan_destroy of a captured plan synchronises the device before its memory is reused.
 * Errors: TN_ERR_DIMENSION (a NULL input, or NULL theta_out[c] for a non-empty slab),
 * TN_ERR_CUDA (launch failure, or a sticky error from earlier work). */
TN_API tn_status tn_theta_exec(const tn_plan* plan, tn_stream stream,
                        const double* gamma_k, const double* lambda_k, const double* gamma_k1,
                        const double* lambda_l, const double* lambda_r, const double* U,
                        double* const* theta_out);

/* ------------------------------------------------------------------------------------------ */
/* SVD step after Θ: PAPER.md:67.                      */
/* ------------------------------------------------------------------------------------------ */
/* tn_svd_truncate — per-sector SVD Θ(c) = U_c diag(s_c) V_c† (default: Gram eigensolver + Rayleigh–Ritz,
 * accurate to rounding for every value that can enter the top χ; TN_SVD_ALGO=gesvdp /
 * gesvdj select a full cuSOLVER SVD per sector), global ranking of
 * every singular value (value descending, then charge ascending, then index ascending),
 * keep the first min(chi_max, #{s > cutoff}) (SPEC.md:98 uses cutoff 1e−14), and write the new
 * canonical factors of bond k (Vidal form, R21): the new bond is ordered by charge
 * ascending, then value descending; for new bond a ↔ (c, s):
 *   q_new[a] = c,  lambda_new[a] = s_c[s]  (not renormalised),
 *   gamma_k_new [α × a] (complex, row-major, ld = *chi_out, rows in the CALLER's α_{k−1} order)
 *                  = U_c[α, s] / λ^{[k−1]}[α] for α in Θ(c)'s rows, 0 elsewhere (x/0 := 0),
 *   gamma_k1_new[a × β] (complex, row-major, ld = χ_r, columns in the caller's α_{k+1} order)
 *                  = V_c†[s, β] / λ^{[k+1]}[β] for β in Θ(c)'s columns, 0 elsewhere.
 *   theta      HOST array of N+1 DEVICE sector pointers from tn_theta_exec — read only (every
 *              path factorises a copy or a projection; Θ(c) is left intact).
 *   lambda_l, lambda_r  DEVICE λ^{[k−1]}, λ^{[k+1]} (the ones passed to tn_theta_exec).
 *   q_new [chi_max] int32, lambda_new [chi_max] double, gamma_k_new [χ_l·chi_max] and
 *   gamma_k1_new [chi_max·χ_r] complex: DEVICE, caller-owned capacity; the factors are written
 *   compact for χ_new = *chi_out (Γk_new is χ_l × χ_new, Γk1_new is χ_new × χ_r), the rest is
 *   unspecified. *chi_out (HOST) = number kept, *discarded (HOST) = Σ of dropped s².
 * MPO pair plans (tn_theta2_plan): the sectors are Θ(c1,c2) (index c1·(N+1)+c2, the
 * ranking's charge order), q_new holds the pair key c1·(N+1)+c2, and Θ(c1,c2)'s rows/columns are its
 * admissible pair segments in sorted order (the layout tn_theta_exec wrote).
 * Synchronises the stream a few times (the kept count is needed on the host). Single-GPU plans only.
 * Errors: TN_ERR_DIMENSION (NULL), TN_ERR_DOMAIN (chi_max < 1, cutoff < 0), TN_ERR_UNSUPPORTED
 * (sharded plan), TN_ERR_OOM, TN_ERR_CUDA (incl. SVD non-convergence). */
TN_API tn_status tn_svd_truncate(const tn_plan* plan, tn_stream stream, double* const* theta,
                                 const double* lambda_l, const double* lambda_r, int64_t chi_max,
                                 double cutoff, int32_t* q_new, double* lambda_new, double* gamma_k_new,
                                 double* gamma_k1_new, int64_t* chi_out, double* discarded);

/* tn_svd_truncate_bform — the same step for an MPS kept in right-canonical ("B") form, B^{[k]} = Γ^{[k]}λ^{[k+1]}
 * (Hastings, J. Math. Phys. 50, 095207 (2009); R22). The caller builds Θ(c) = λ^{[k−1]} B^{[k]} B^{[k+1]}
 * (gated) with tn_theta_exec(gamma_k = B^{[k]}, lambda_k = 1, gamma_k1 = B^{[k+1]}, lambda_l = λ^{[k−1]},
 * lambda_r = 1); ranking, q_new and lambda_new are as tn_svd_truncate's, and the new factors need no division by a
 * singular value or a small λ:
 *   b_k_new  [χ_l × χ_new] (ld *chi_out): B^{[k]}_new[α, a]  = (Θ(c)·V_c)[α, s] / λ^{[k−1]}[α]  (undoes Θ's own row
 *            scaling, exact to rounding per element; x/0 := 0)
 *   b_k1_new [χ_new × χ_r]:              B^{[k+1]}_new[a, β] = V_c†[s, β]
 * Arguments, synchronisation and errors as tn_svd_truncate (lambda_r is not needed). */
TN_API tn_status tn_svd_truncate_bform(const tn_plan* plan, tn_stream stream, double* const* theta,
                                       const double* lambda_l, int64_t chi_max, double cutoff, int32_t* q_new,
                                       double* lambda_new, double* b_k_new, double* b_k1_new, int64_t* chi_out,
                                       double* discarded);

/* ------------------------------------------------------------------------------------------ */
/* Multi-GPU (one process per GPU): row-sharded exec + NCCL.                 */
/* ------------------------------------------------------------------------------------------ */
/* 128-byte NCCL unique id for rank 0 to create and distribute (e.g. via torch.distributed). */
TN_API tn_status tn_comm_unique_id(void* id128);
/* Bootstrap a communicator; NCCL is loaded at run time (dlopen "libnccl.so.2", or $TN_NCCL_LIB). */
TN_API tn_status tn_comm_init(const void* id128, int rank, int world_size, tn_comm** out);
TN_API tn_status tn_comm_destroy(tn_comm* comm);
/* Where rank `rank`'s slab of sector c lies inside the FULL Θ(c): its first row and row count (HOST
 * outputs; what the ROOT / SECTOR_OWNER gathers use to place each rank's rows, for single-charge and
 * pair plans). Errors: DIMENSION (NULL), DOMAIN (c or rank out of range). */
TN_API tn_status tn_plan_slab_rows(const tn_plan* plan, int c, int rank, int64_t* row_begin, int64_t* rows);

/* The exact transfer list tn_theta_exec_sharded executes for gather_mode: one entry per
 * (sector, source rank) with a non-empty slab, sectors ascending then source rank ascending, destination
 * rank 0 (TN_GATHER_ROOT) or tn_plan_sector_owner(sector) (TN_GATHER_SECTOR_OWNER); none for
 * TN_GATHER_NONE. Identical on every rank. HOST outputs: *n_out = number of entries; the first
 * min(capacity, *n_out) are written to out (out may be NULL with capacity 0 to query the count).
 * Errors: DIMENSION (NULL plan/n_out, or capacity < *n_out with out != NULL), DOMAIN (gather_mode). */
TN_API tn_status tn_plan_gather_schedule(const tn_plan* plan, int gather_mode, int64_t capacity, tn_transfer* out,
                                         int64_t* n_out);
/* The same schedule without a plan or a GPU (single-charge layout, R2): from host offset tables
 * off_l / off_r (N+2 int32 each, as tn_plan_offsets returns) and row-shard bounds (world_size+1 int64, as
 * tn_shard_rows_host returns); sector owners by the tn_sector_owners_host rule. Errors as above, plus
 * DOMAIN for decreasing offsets or bounds. */
TN_API tn_status tn_gather_schedule_host(int d, int N, const int32_t* off_l, const int32_t* off_r, int world_size,
                                         const int64_t* bounds, int gather_mode, int64_t capacity,
                                         tn_transfer* out, int64_t* n_out);
/* The communicator's asynchronous error state (ncclCommGetAsyncError): TN_OK, or TN_ERR_NCCL with the NCCL
 * error in tn_last_error(). tn_theta_exec_sharded checks it before and after each grouped call. */
TN_API tn_status tn_comm_async_error(tn_comm* comm);

/* Row-slab operands (the TN_BCAST_SLABS distribution, usable on its own when the caller moves the slabs):
 * tn_pack_row_slab writes rank `rank`'s rows of Γk — sorted left positions [r0, r1) of that rank's shard
 * (tn_plan_shard_rows) — packed in sorted order: slab_out[(p − r0)·χ_c + k] = Γk[perm_l[p]][k]
 * (K6 `k6_pack_rows`; gamma_k DEVICE complex [χ_l × χ_c] caller order, slab_out DEVICE complex of
 * (r1−r0)·χ_c entries, caller-owned). tn_theta_exec_slab is tn_theta_exec for the plan's own rank with Γk
 * given as that packed slab (gamma_k_slab; every other argument as tn_theta_exec), so a rank never holds
 * the rows of other shards. Stream-ordered, no host sync. Errors: DIMENSION (NULL), DOMAIN (rank),
 * UNSUPPORTED (the paper-literal ablation engine), CUDA. */
TN_API tn_status tn_pack_row_slab(const tn_plan* plan, tn_stream stream, const double* gamma_k, int rank,
                                  double* slab_out);
TN_API tn_status tn_theta_exec_slab(const tn_plan* plan, tn_stream stream, const double* gamma_k_slab,
                                    const double* lambda_k, const double* gamma_k1, const double* lambda_l,
                                    const double* lambda_r, const double* U, double* const* theta_out);

/* tn_theta_exec_sharded — this rank's rows of every Θ(c), plus optional exchange.
 *   plan          built with the communicator's world_size and rank (else TN_ERR_CONSISTENCY).
 *   bcast_operands operand distribution from rank 0 before the compute:
 *                 TN_BCAST_NONE  — every rank already holds its operands (full-size, caller order).
 *                 TN_BCAST_SLABS — rank 0 holds Γk (caller order); each other rank receives ONLY its row
 *                   slab: rank 0 packs the other ranks' rows in sorted order (tn_pack_row_slab's K6) and
 *                   sends each rank its run, which lands in gamma_k as the packed (r1−r0) × χ_c slab
 *                   (gamma_k needs only that capacity on ranks > 0) and is consumed as by
 *                   tn_theta_exec_slab. Γk1, λk, λl, λr and U — replicated by design — are
 *                   ncclBroadcast into the same full-size buffers on every rank.
 *                 TN_BCAST_FULL  — the whole Γk is broadcast as well (every rank full-size, caller order).
 *   gather_mode   TN_GATHER_NONE: theta_out holds the local slabs (tn_plan_local_sector_shape).
 *                 TN_GATHER_ROOT: on rank 0 theta_out holds the FULL Θ(c) (R_c×C_c) and every
 *                 rank's slab is sent to it with grouped ncclSend/ncclRecv; on other ranks
 *                 theta_out holds the local slabs.
 *                 TN_GATHER_SECTOR_OWNER: Θ(c) goes to rank tn_plan_sector_owner(c)
 *                 (sectors spread over ranks by element count — the hand-off to per-sector SVD); on the
 *                 owner theta_out[c] holds the FULL Θ(c), elsewhere the local slab.
 *                 The transfers are exactly tn_plan_gather_schedule(plan, gather_mode).
 * Other arguments as tn_theta_exec. Errors: as tn_theta_exec, plus TN_ERR_NCCL (including an asynchronous
 * communicator error), TN_ERR_CONSISTENCY, TN_ERR_DOMAIN (unknown mode), TN_ERR_UNSUPPORTED (TN_BCAST_SLABS
 * with the paper-literal ablation engine). */
TN_API tn_status tn_theta_exec_sharded(const tn_plan* plan, tn_stream stream, tn_comm* comm,
                                double* gamma_k, double* lambda_k, double* gamma_k1,
                                double* lambda_l, double* lambda_r, double* U,
                                double* const* theta_out, int bcast_operands, int gather_mode);

/* tn_theta_exec_remote — the SECTOR_OWNER exchange fused into the computation (SURVEY.md §8(e)
 * "Optional fusion"): K4 writes this rank's P into a plan-owned LOCAL workspace, and K5 writes each row
 * of this rank's slab of Θ(c) straight to theta_dst[c] — any device-accessible pointer, typically the
 * owner rank's full Θ(c) buffer opened with tn_ipc_open (NVLink peer memory) offset to this rank's
 * first row (tn_plan_local_sector_shape's row_begin × C_c complex). No collective runs inside: the
 * caller orders consumers after every rank's stream (e.g. a barrier after synchronising). Other
 * arguments as tn_theta_exec. Single-charge and MPO pair plans (K5P: first pass in place on the local
 * workspace, second pass into theta_dst) with the DMMA or INT8 engine; TN_ERR_UNSUPPORTED otherwise. */
TN_API tn_status tn_theta_exec_remote(tn_plan* plan, tn_stream stream, const double* gamma_k,
                                      const double* lambda_k, const double* gamma_k1, const double* lambda_l,
                                      const double* lambda_r, const double* U, double* const* theta_dst);
/* CUDA IPC for tn_theta_exec_remote: 64-byte handle + byte offset of dev_ptr inside its allocation;
 * open a peer process's handle (peer access enabled lazily); close what tn_ipc_open returned. */
TN_API tn_status tn_ipc_get_handle(const void* dev_ptr, void* handle64, int64_t* offset);
TN_API tn_status tn_ipc_open(const void* handle64, void** dev_ptr);
TN_API tn_status tn_ipc_close(void* dev_ptr);

/* ------------------------------------------------------------------------------------------ */
/* Host-only helpers (no GPU needed) and diagnostics.                                          */
/* ------------------------------------------------------------------------------------------ */
/* Flop-balanced row shards from per-charge bond counts n_x[0..N] (the plan's own rule):
 * bounds[0..world_size] (world_size+1 int64) of sorted left positions, bounds[0]=0,
 * bounds[world_size]=χ_l. Errors: TN_ERR_DOMAIN. */
TN_API tn_status tn_shard_rows_host(int d, int N, const int64_t* n_l, const int64_t* n_c,
                             const int64_t* n_r, int world_size, int64_t* bounds);
/* The plan's sector-owner rule on host data: owners[0..n_sectors) from element counts sizes[]. */
TN_API tn_status tn_sector_owners_host(int n_sectors, const int64_t* sizes, int world_size, int32_t* owners);

/* Device memory: plan tables and staging workspace come from a library-owned pool. A destroyed
 * plan's blocks are reused by later plans once the work last enqueued with them has completed
 * (an event recorded on the last exec stream), so per-gate planning does not call cudaMalloc.
 * tn_release_cached_memory frees every idle block (waiting for its event) and reports the bytes
 * freed; *cached (may be NULL) receives the bytes still held by live plans. */
TN_API tn_status tn_release_cached_memory(int64_t* freed, int64_t* cached);

/* Pipelined gates: makes the pool hold at least `count` blocks (in use or idle) of each size `plan`
 * holds (tables, workspace and any exec_sharded / INT8 / literal workspace created so far), allocating
 * the missing ones now. A caller that keeps up to `count` plans of this shape alive at once (gates in
 * flight on several streams, plans kept for kernel_times) then never reaches cudaMalloc on the
 * enqueue path: a cudaMalloc of a workspace-sized block costs the host milliseconds, during which
 * the GPU drains its queue. New blocks are sized with ≤ 6.25% slack so that plans of slightly
 * different shape share them. count ≤ 0 is a no-op. Errors: TN_ERR_CUDA (out of memory; the blocks
 * allocated before the failure stay in the pool). */
TN_API tn_status tn_plan_reserve(const tn_plan* plan, int32_t count);

TN_API const char* tn_status_string(tn_status s);
TN_API const char* tn_last_error(void);       /* thread-local detail of the last failure ("" if none) */
TN_API int tn_version(void);                  /* (major << 16) | minor */

#ifdef __cplusplus
}
#endif
#endif /* TN_THETA_H */
