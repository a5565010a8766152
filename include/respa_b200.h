/*
 * respa_b200.h -- C-ABI of the B200 (sm_100a) force-evaluation hot path for
 * the arXiv 2507.11172 reference engine (LJ + Axilrod-Teller-Muto with
 * r-RESPA multiple time-stepping).
 *
 * The reference ("respamd", pure Python + numba) has no FFI: its hot path is
 * reached through the container duck type (pair_pass / triplet_pass,
 * respamd/containers.py:878-937), the functional passes
 * (build_cell_grid :235, c01_pair_pass :750, c01_triplet_pass :786,
 * collect_triplet_visits :825) and respa_run (respamd/integrators.py:96-173).
 * Each entry point below replaces the numba kernel named beside it; the
 * Python mirror (paper_2507_11172_b200/, binding shown in INTEGRATION.md)
 * calls them through ctypes.
 *
 * Conventions
 *   - all array arguments are DEVICE pointers (cudaMalloc / torch CUDA
 *     tensors) unless stated; per-particle state is the reference layout,
 *     (n,3) float64 AoS in particle order;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - no entry point allocates memory: callers own every buffer; scratch is
 *     sized by the matching *_scratch_bytes query;
 *   - the return value is a launch-time status (RB_OK or RB_ERR_*); data-
 *     dependent errors found on the device (minimum separation, non-finite
 *     state, list overflow) are recorded in a caller-owned device status
 *     word, `unsigned long long *status`, as (tag << 8) | kind by atomicMin.
 *     Initialise it to RB_STATUS_CLEAR.  `tag` is the r-RESPA iteration the
 *     kernel belongs to (0 for standalone passes); a kernel whose tag is
 *     larger than a recorded error's tag does nothing, so the state freezes
 *     at the failing step as respamd's IntegrationBlowUp does.  The device
 *     loop uses four words (error, current step, last closed step, rebuild
 *     steps); the array must be 16-byte aligned (read in word pairs).
 */
#ifndef RESPA_B200_H
#define RESPA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define RB_API __attribute__((visibility("default")))
#else
#define RB_API
#endif

#define RB_ABI_VERSION 1

/* return / status kinds */
#define RB_OK 0
#define RB_ERR_MIN_SEPARATION 1 /* respamd MinimumSeparationError (containers.py:39-40,742-747) */
#define RB_ERR_GEOMETRY 2       /* respamd ValidationError for the grid (containers.py:248-252) */
#define RB_ERR_CUDA 3           /* launch failure */
#define RB_ERR_CAPACITY 4       /* a neighbour row exceeded its capacity */
#define RB_ERR_ARGUMENT 5       /* bad sizes or pointers */
#define RB_NOT_CAPTURING 6      /* rb_rebuild_cond_begin outside a stream capture */

/* device status-word kinds (low 8 bits), ordered by precedence inside a step */
#define RB_KIND_PAIR_MIN_SEPARATION 1    /* raised by pair_pass (integrators.py:154-157) */
#define RB_KIND_TRIPLET_MIN_SEPARATION 2 /* raised by triplet_pass (:161-164) */
#define RB_KIND_NONFINITE 3              /* _check_finite (:89-93, :166-170) */
#define RB_KIND_CAPACITY 4               /* neighbour-list overflow (no reference analogue) */
#define RB_KIND_REBUILD 0                /* not an error: a rebuild vote froze the steps from
                                            `tag` on (speculative windows of the decomposed
                                            loop, rb_vote_freeze); drift, kick, sample and the
                                            halo pull stop too, so the host rebuilds and
                                            resumes step `tag` */
#define RB_STATUS_CLEAR 0xFFFFFFFFFFFFFFFFull

#define RB_MAX_OFFSETS 125

/* Cell-grid geometry, computed on the host exactly as
 * respamd/containers.py:244-263 does (cells = max(1, floor(extent/cutoff)),
 * size = extent/cells, inv_cell = 1.0/size) so that binning is bit-exact. */
typedef struct rb_grid {
    int32_t cells[3];   /* cells per dimension (local cells when windowed) */
    int32_t periodic;   /* 1: periodic box with single-shift minimum image */
    double origin[3];   /* 0 for periodic systems */
    double inv_cell[3]; /* 1.0 / cell_size */
    double box[3];
    int32_t n_offsets;                   /* canonical neighbour-cell offsets */
    int32_t offsets[RB_MAX_OFFSETS][3];  /* containers.py:133-144 (pair_cells) */
    /* Domain decomposition (rb_grid_window): per dimension, wrap[d] = 1 when
     * neighbour-cell indices wrap (whole periodic dimension), 0 when the
     * local grid is a window [wlo, wlo + cells) of the global periodic grid
     * of gcells cells (a rank's block plus one halo layer); binning maps the
     * global cell index into the window.  Distances always use the periodic
     * minimum image of the whole box, so predicates stay bit-exact. */
    int32_t wrap[3];
    int32_t gcells[3];
    int32_t wlo[3];
} rb_grid;

RB_API int rb_abi_version(void);
/* cumulative number of kernels this library has launched (or recorded into
 * a CUDA graph under capture) in this process */
RB_API long long rb_launch_count(void);
/* sizeof(rb_grid) as compiled into the library (binding layout check) */
RB_API size_t rb_grid_bytes(void);
RB_API const char *rb_status_string(int status);
/* number of CUDA devices visible to this library's runtime (0 without a GPU) */
RB_API int rb_device_count(void);

/* ---- binning: replaces _bin_particles (containers.py:175-209) ----------
 * Counting sort of particles by flat cell id (cx*ny+cy)*nz+cz with the
 * truncating index of :182-197, stable in ascending particle index.
 * Outputs: cell_start[ncell+1], cell_particles[n] (rank -> particle),
 * cell_of_rank[n], and positions gathered into rank order, pos_r (n,3) --
 * the layout every force pass reads (one 24-byte gather per neighbour). */
RB_API size_t rb_bin_scratch_bytes(int64_t n, int64_t ncell);
/* rank_of[n] (particle -> rank) and x_ref (n,3) (positions at this build)
 * are optional (NULL).  rebuild_flag gates the launch for captured
 * r-RESPA steps: the kernels run only when *rebuild_flag equals the step
 * tag (see rb_respa_drift); NULL = always. */
RB_API int rb_bin(const rb_grid *g, int64_t n, const double *pos, int32_t *cell_start,
                  int32_t *cell_particles, int32_t *cell_of_rank, double *pos_r,
                  int32_t *rank_of, double *x_ref, const int64_t *rebuild_flag,
                  const unsigned long long *status, int64_t tag, void *scratch,
                  size_t scratch_bytes, void *stream);

/* ---- neighbour rows: the survivor lists of containers.py:437-474 -------
 * Row r (rank order) lists, in stencil order, the ranks within r_list of
 * particle r (reference pair-distance arithmetic, inclusive).  Rows hold at
 * most `capacity` entries; the longest row length is atomicMax-ed into the
 * device int *max_count (caller initialises it to 0).  A row longer than
 * `capacity` is truncated, so callers must check *max_count <= capacity
 * before trusting a pass. */
RB_API int rb_nlist(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_start,
                    const int32_t *cell_of_rank, double r_list, int32_t capacity, int32_t *rows,
                    int32_t *row_count, int32_t *max_count, const int64_t *rebuild_flag,
                    const unsigned long long *status, int64_t tag, void *stream);

/* ---- LJ pair pass: replaces _c01_pair_kernel (containers.py:282-370) ---
 * Owner-computes over the neighbour rows with the inclusive cutoff `rc`;
 * writes forces (n,3) in particle order (overwritten), and per-rank energy
 * (sum of phi/2) and virial (sum of scale*r^2/2).  `owned` (rank-indexed,
 * NULL = all) zeroes the energy/virial of ghost particles in decomposed runs. */
RB_API int rb_lj_pass(const rb_grid *g, int64_t n, const double *pos_r,
               const int32_t *cell_particles, const int32_t *rows, const int32_t *row_count,
               int32_t capacity, double rc, double epsilon, double sigma, double *forces,
               double *energy_rank, double *virial_rank, const uint8_t *owned,
               unsigned long long *status, int64_t tag, void *stream);

/* Mirror indices of the (rank-sorted) rows: mirror[p*capacity + k] is the
 * position of p in the row of q = rows[p*capacity + k], written for the
 * entries with q > p only (the others are left as they were; -1: p is not
 * in row q, a truncated row).  The Newton-3 triplet pass uses it to deliver
 * partial forces into the target's row. */
RB_API int rb_nlist_mirror(int64_t n, const int32_t *rows, const int32_t *row_count,
                           int32_t capacity, int32_t *mirror, const int64_t *rebuild_flag,
                           const unsigned long long *status, int64_t tag, void *stream);

/* Rows and their mirror in one call: rb_nlist's rows, then rb_nlist_mirror's
 * entries (the same values).  On grids the cell-staged row build serves
 * (>= 4 cells per periodic dimension) the mirror comes from the cell
 * structure instead of a search: the row build writes per-row directories
 * (survivors before each neighbour cell) and per-entry partials, and one
 * pass adds them.  scratch: rb_nlist_mirror_scratch_bytes(n) bytes, any
 * contents. */
RB_API size_t rb_nlist_mirror_scratch_bytes(int64_t n);
RB_API int rb_nlist_rows_mirror(const rb_grid *g, int64_t n, const double *pos_r,
                                const int32_t *cell_start, const int32_t *cell_of_rank,
                                double r_list, int32_t capacity, int32_t *rows,
                                int32_t *row_count, int32_t *max_count, int32_t *mirror,
                                void *scratch, size_t scratch_bytes,
                                const int64_t *rebuild_flag, const unsigned long long *status,
                                int64_t tag, void *stream);

/* ---- ATM triplet pass: replaces _c01_triplet_kernel (:373-535) --------
 * Newton-3 form: every unique triplet (all three pair distances <= rc,
 * inclusive, reference arithmetic) is evaluated once by its lowest-rank
 * member; forces on all three members are accumulated without atomics in a
 * fixed order (deterministic).  Writes forces (n,3) in particle order
 * (overwritten), per-rank energy (phi per owned triplet), virial and the
 * number of owned (unique) triplets.  Scratch: rb_atm_scratch_bytes,
 * zero-filled before its first use (each pass leaves its work counter and
 * overflow-list count at zero; they sit at fixed offsets, so one scratch
 * serves passes of any n up to the size it was made for).  Persistent warps
 * take the bases from a work counter (RB_ATM_PERSIST=0: one base per warp).  slot_capacity (<= capacity) sizes the per-warp
 * shared-memory slots; a particle with more higher-rank neighbours than
 * that records RB_KIND_CAPACITY in the status word (pass the longest row
 * length).  The pass runs most particles with about half the slots (higher
 * occupancy) and the few longer S+ sets in a second full-slot launch.
 * `owned` (rank-indexed, NULL = all): in decomposed runs a triplet's
 * energy/virial is weighted by (owned members)/3, the reference's phi/3 per
 * member; forces on ghosts are computed and left to the caller to drop. */
RB_API size_t rb_atm_scratch_bytes(int64_t n, int32_t capacity);
RB_API int rb_atm_pass(const rb_grid *g, int64_t n, const double *pos_r,
                       const int32_t *cell_particles, const int32_t *rows,
                       const int32_t *row_count, const int32_t *mirror, int32_t capacity,
                       int32_t slot_capacity, double rc, double nu, double *forces,
                       double *energy_rank, double *virial_rank, int32_t *triplets_rank,
                       const uint8_t *owned, void *scratch, size_t scratch_bytes,
                       unsigned long long *status, int64_t tag, void *stream);
/* The same pass in two stream-ordered parts (part 0 = both = rb_atm_pass):
 * part 1 launches the triplet kernels, whose results stay in the scratch;
 * part 2 the gather, which alone writes forces, energy_rank, virial_rank and
 * triplets_rank.  Between them the caller may run the pair pass on another
 * stream (the device loop overlaps it with the tail of part 1); a pair-pass
 * error of the same step then still leaves the triplet outputs untouched.
 * Every part 1 must be followed by its part 2 (stream-ordered) before the
 * next pass on the same scratch: part 2 also resets the pass's work counter
 * and overflow list. */
RB_API int rb_atm_pass_part(const rb_grid *g, int64_t n, const double *pos_r,
                            const int32_t *cell_particles, const int32_t *rows,
                            const int32_t *row_count, const int32_t *mirror, int32_t capacity,
                            int32_t slot_capacity, double rc, double nu, double *forces,
                            double *energy_rank, double *virial_rank, int32_t *triplets_rank,
                            const uint8_t *owned, void *scratch, size_t scratch_bytes,
                            unsigned long long *status, int64_t tag, int32_t part,
                            void *stream);

/* Cell-based form of the same Newton-3 pass (same results, same outputs):
 * one CTA per base cell stages the stencil cells that can hold the S+ sets
 * of its particles (cells whose index is >= its own) in shared memory,
 * builds S+(i) from them (fp32 filter, reference arithmetic decides), runs
 * the pair loop and reduces the partial forces per target in shared memory;
 * one 32-byte entry per (particle, source cell) goes through the scratch to
 * the gather.  Needs no neighbour rows: `cell_start` (ncell + 1) and
 * `cell_of_rank` from rb_bin.  Supported when rb_atm_cells_supported (reach-1
 * stencil with cell size >= rc, periodic boxes of at least four cutoffs);
 * otherwise use rb_atm_pass_part.  `nb_cap` = staged particles per cell
 * (>= rb_atm_cells_nb_max), `slot_capacity` (32..256) = longest S+(i); a
 * cell or base over either records RB_KIND_CAPACITY.  Scratch:
 * rb_atm_cells_scratch_bytes, zero-filled before first use (part 2 leaves
 * its cell counter at zero).  Parts as rb_atm_pass_part. */
RB_API size_t rb_atm_cells_scratch_bytes(int64_t n);
RB_API size_t rb_atm_cells_smem_bytes(int32_t nb_cap, int32_t slot_capacity);
RB_API int rb_atm_cells_supported(const rb_grid *g, double rc);
RB_API int rb_atm_cells_nb_max(const rb_grid *g, const int32_t *cell_start, int32_t *out,
                               void *stream);
RB_API int rb_atm_pass_cells(const rb_grid *g, int64_t n, const double *pos_r,
                             const int32_t *cell_particles, const int32_t *cell_start,
                             const int32_t *cell_of_rank, int32_t nb_cap, int32_t slot_capacity,
                             double rc, double nu, double *forces, double *energy_rank,
                             double *virial_rank, int32_t *triplets_rank, const uint8_t *owned,
                             void *scratch, size_t scratch_bytes, unsigned long long *status,
                             int64_t tag, int32_t part, void *stream);

/* C01 (owner-computes) form of the same pass, as the reference traverses it:
 * every triplet visited once from each member, force stored on the base
 * particle only, energy phi/3 per visit; visits_rank = accepted visits. */
RB_API int rb_atm_pass_c01(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_particles, const int32_t *rows,
                           const int32_t *row_count, int32_t capacity, double rc, double nu,
                           double *forces, double *energy_rank, double *virial_rank,
                           int32_t *visits_rank, unsigned long long *status, int64_t tag,
                           void *stream);

/* Instrumentation (collect_triplet_visits, containers.py:825-849): writes
 * one sorted (i, j, k) particle-index row per accepted visit, int32 (V,3),
 * at row_offset[r] (exclusive prefix of rb_atm_pass_c01's visits_rank). */
RB_API int rb_atm_visit_rows(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_particles, const int32_t *rows,
                             const int32_t *row_count, int32_t capacity, double rc,
                             const int64_t *row_offset, int32_t *visit_rows, void *stream);

/* ---- DirectSum: replaces _direct_pair_kernel / _direct_triplet_kernel
 * (containers.py:663-739) -- all pairs / all triplets of a NON-periodic
 * system, no cutoff, the reference's raw differences and guard.
 * rb_direct_pairs: forces (n,3) in particle order (overwritten) and the
 *   per-particle halves of the pair energy and virial (sum them with
 *   rb_reduce_sum_f64); owner-computes, deterministic.
 * rb_direct_triplets: Newton-3, forces (n,3) (overwritten) and
 *   energy_virial[2] = (E3, W3) on the device; n <= 8192; scratch
 *   rb_direct_scratch_bytes(n); deterministic (fixed block partition and
 *   block-order sums). */
RB_API int rb_direct_pairs(int64_t n, const double *pos, double epsilon, double sigma,
                           double *forces, double *energy_part, double *virial_part,
                           unsigned long long *status, int64_t tag, void *stream);
RB_API size_t rb_direct_scratch_bytes(int64_t n);
RB_API int rb_direct_triplets(int64_t n, const double *pos, double nu, double *forces,
                              double *energy_virial, void *scratch, size_t scratch_bytes,
                              unsigned long long *status, int64_t tag, void *stream);
/* The share of one rank of a distributed DirectSum: rb_direct_pairs_range
 * writes forces / energy halves of the particles [i_lo, i_hi) only;
 * rb_direct_triplets_range evaluates the triplets whose lowest member is in
 * [i_lo, i_hi) and writes their forces on ALL particles (overwritten) and
 * their (E3, W3).  Summed over ranks covering [0, n) the parts give the full
 * pass. */
RB_API int rb_direct_pairs_range(int64_t n, const double *pos, int64_t i_lo, int64_t i_hi,
                                 double epsilon, double sigma, double *forces,
                                 double *energy_part, double *virial_part,
                                 unsigned long long *status, int64_t tag, void *stream);
RB_API int rb_direct_triplets_range(int64_t n, const double *pos, int64_t i_lo, int64_t i_hi,
                                    double nu, double *forces, double *energy_virial,
                                    void *scratch, size_t scratch_bytes,
                                    unsigned long long *status, int64_t tag, void *stream);

/* ---- radial distribution function: replaces _distance_histogram
 * (observables.py:143-177).  counts[bins] (int64, device) += ordered
 * minimum-image pair counts with r^2 < r2_max in bin
 * trunc(sqrt(r^2) * inv_width) (clamped); pass r2_max = r_max * r_max and
 * inv_width = bins / r_max computed as the reference does.  Bit-exact
 * integer counts. */
RB_API int rb_distance_histogram(int64_t n, const double *pos, const double *box3_host,
                                 double r2_max, double inv_width, int32_t bins, int64_t *counts,
                                 void *stream);

/* ---- halo exchange of the domain-decomposed loop ------
 * rb_halo_pack: buf[i] = pos[idx[i]] (24-byte records), the message of one
 * send list.  rb_halo_unpack: pos[first + i] = buf[i] for a received
 * message of n ghosts and, with pos_r != NULL, the rank-ordered copy
 * pos_r[rank_of[first + i]].  The messages themselves travel over NCCL
 * (torch.distributed point-to-point) between the two calls. */
RB_API int rb_halo_pack(int64_t n, const int32_t *idx, const double *pos, double *buf,
                        void *stream);
RB_API int rb_halo_unpack(int64_t n, const double *buf, int64_t first, double *pos,
                          const int32_t *rank_of, double *pos_r, void *stream);

/* Peer-memory form (no messages): each rank publishes its owned positions
 * from the step's drift (rb_respa_drift_publish, advance_step only: row p
 * of the half (tag & 1) of `publish`, halves `stride` rows apart, then a
 * system-scope fence) into one IPC-shared allocation; after the step's
 * rebuild vote (which orders every rank's drift before every rank's pull),
 * rb_halo_pull reads ghost row first + i from row src_index[i] of the half
 * (status[1] & 1) of peers[src_rank[i]] (device array of the ranks' mapped
 * base pointers, all with the same `stride`) into pos and, with
 * pos_r != NULL, pos_r[rank_of[first + i]].  The parity comes from the
 * device step counter, so a captured step replays at either parity.
 * Bit-identical to pack / send / unpack. */
RB_API int rb_respa_drift_publish(int64_t n, double *pos, double *vel, const double *f2_old,
                                  const double *f3, const double *box3_host, int32_t periodic,
                                  double dt, double half_drift, double half_respa, int32_t kick3,
                                  const int32_t *rank_of, double *pos_r, const double *x_ref,
                                  double skin, int64_t *rebuild_flag, unsigned long long *status,
                                  int64_t tag, int32_t advance_step, double *publish,
                                  int64_t stride, void *stream);
RB_API int rb_halo_pull(int64_t n, const int32_t *src_rank, const int32_t *src_index,
                        const uint64_t *peers, int64_t stride, const unsigned long long *status,
                        int64_t first, double *pos, const int32_t *rank_of, double *pos_r,
                        void *stream);
/* CUDA IPC: a cudaMalloc'd (zeroed) allocation, its 64-byte handle, and the
 * peer-side mapping (cudaIpcMemLazyEnablePeerAccess) / unmapping. */
RB_API int rb_ipc_alloc(int64_t bytes, void **ptr);
RB_API int rb_ipc_free(void *ptr);
RB_API int rb_ipc_handle(void *ptr, uint8_t *handle64);
RB_API int rb_ipc_open(const uint8_t *handle64, void **ptr);
RB_API int rb_ipc_close(void *ptr);

/* ---- deterministic reductions (fixed partition + fixed tree) ---------- */
RB_API size_t rb_reduce_scratch_bytes(int64_t n);
/* out[0] = sum(in[0..n)) */
RB_API int rb_reduce_sum_f64(int64_t n, const double *in, double *out, void *scratch, void *stream);
/* out[0] = sum(in[i]^2) -- kinetic energy numerator of model.py:133 */
RB_API int rb_reduce_sumsq_f64(int64_t n, const double *in, double *out, void *scratch, void *stream);
/* out[0] = sum(in[0..n)) as int64 */
RB_API int rb_reduce_sum_i32(int64_t n, const int32_t *in, int64_t *out, void *scratch, void *stream);

/* ---- r-RESPA kick/drift: replaces the numpy updates of respa_run ------
 * (integrators.py:148-170), bit-exact with numpy's rounding order.
 * drift: [v += half_respa*f3 if kick3]; x += dt*v + half_drift*f2_old;
 *        wrap into [0, box) with numpy mod semantics (model.py:274-280);
 *        non-finite x records RB_KIND_NONFINITE at `tag`.  Optionally
 *        (non-NULL) scatters x into pos_r via rank_of, and sets
 *        *rebuild_flag = tag when a particle moved more than skin/2 from
 *        x_ref (the neighbour rows, built at rc + skin, must be rebuilt).
 *        advance_step != 0 (tag must be -1): the drift opens a new device
 *        step -- its tag is status[2] + 1 (the last closed step + 1) and it
 *        writes it to status[1] for the step's later kernels; the step's
 *        kick (tag -1) closes it.  rebuild_cond != 0: a CUDA-graph
 *        conditional handle (rb_rebuild_cond_create) set to 1 together with
 *        the rebuild flag.
 * kick:  v += half_dt*(f2_old + f2_new); f2_old = f2_new (:159);
 *        [v += half_respa*f3 if kick3];
 *        non-finite v records RB_KIND_NONFINITE at `tag`. */
RB_API int rb_respa_drift(int64_t n, double *pos, double *vel, const double *f2_old,
                          const double *f3, const double *box3_host, int32_t periodic, double dt,
                          double half_drift, double half_respa, int32_t kick3,
                          const int32_t *rank_of, double *pos_r, const double *x_ref,
                          double skin, int64_t *rebuild_flag, unsigned long long *status,
                          int64_t tag, int32_t advance_step, uint64_t rebuild_cond,
                          void *stream);
/* The kick that ends step i-1 folded into the drift that opens step i (one
 * pass over the particles): v += half_dt (f2_old + f2_new) [+ half_respa f3
 * if kick3_prev]; f2_old = f2_new -- with rb_respa_kick's error rules at
 * tag i-1 -- then the step-opening drift of rb_respa_drift (advance_step,
 * tags from the device) with kick3 at cycle start.  Bit-identical to the two
 * launches. */
RB_API int rb_respa_kick_drift(int64_t n, double *pos, double *vel, double *f2_old,
                               const double *f2_new, const double *f3, const double *box3_host,
                               int32_t periodic, double dt, double half_dt, double half_drift,
                               double half_respa, int32_t kick3_prev, int32_t kick3,
                               const int32_t *rank_of, double *pos_r, const double *x_ref,
                               double skin, int64_t *rebuild_flag, unsigned long long *status,
                               uint64_t rebuild_cond, void *stream);
/* Speculative windows of the decomposed loop: the rebuild
 * vote of the current device step without a host round trip.
 * rb_vote_flag:   *flag = 1 if this rank's drift flagged the current step
 *                 (rebuild_flag[0] == status[1]), else 0 -- the input of an
 *                 all_reduce(MAX) over the ranks (captured with the step);
 * rb_vote_freeze: if *flag > 0 and no error is recorded, records
 *                 RB_KIND_REBUILD at the current step: every later kernel of
 *                 the window exits, the host reads the word once per window.
 * Replace the per-step host vote of the reference-less multi-GPU loop; no
 * reference analogue (the reference's distributed mode is out of scope,
 * SPEC.md:13). */
RB_API int rb_vote_flag(const int64_t *rebuild_flag, const unsigned long long *status,
                        int64_t *flag, void *stream);
RB_API int rb_vote_freeze(const int64_t *flag, unsigned long long *status, void *stream);

RB_API int rb_respa_kick(int64_t n, double *vel, double *f2_old, const double *f2_new,
                  const double *f3, double half_dt, double half_respa, int32_t kick3,
                  unsigned long long *status, int64_t tag, void *stream);

/* ---- device-side step counter and trace (CUDA-graph friendly) ---------
 * status points to FOUR words: status[0] the error word, status[1] the
 * current step, status[2] the last closed step, status[3] the number of
 * steps in which a drift flagged a row rebuild (diagnostic).  A
 * step-opening drift (advance_step) numbers its step status[2] + 1 and
 * writes it to status[1]; the step's pair pass and kick with tag -1 close it
 * (status[2] = status[1]); rb_step_begin does both in one launch (status[2] =
 * status[1], status[1] += 1).  Kernels given tag == -1 read their tag from status[1].
 * rb_step_begin increments status[1]; rb_trace_record writes the 8-double
 * row [tag, sum v^2, E2, W2, E3, W3, 0, 0] at trace[8 * (tag / interval)]
 * from device scalars (RunTrace.record, integrators.py:74-83). */
RB_API int rb_step_begin(unsigned long long *status, void *stream);
RB_API int rb_trace_record(const unsigned long long *status, int64_t sample_interval,
                           double *trace, const double *sumsq, const double *e2, const double *w2,
                           const double *e3, const double *w3, void *stream);

/* ---- conditional rebuild inside a captured step (CUDA graph IF node) ----
 * In a CUDA-graph capture the gated rebuild (rb_bin, rb_nlist,
 * rb_nlist_mirror with rebuild_flag set) would cost nine launches per step
 * even when its gate is closed.  rb_rebuild_cond_create makes a conditional
 * handle in the graph `stream` is capturing into (RB_NOT_CAPTURING outside
 * a capture: launch the gated kernels directly, results are identical); it
 * is passed to rb_respa_drift, which sets it with the rebuild flag.
 * rb_rebuild_cond_begin appends the IF node on that handle and returns in
 * *body_stream a stream capturing into its body: launch the gated rebuild
 * there, then rb_rebuild_cond_end(stream) continues the capture after the
 * node.  One conditional may be open per host thread. */
RB_API int rb_rebuild_cond_create(void *stream, uint64_t *handle);
RB_API int rb_rebuild_cond_begin(uint64_t handle, void *stream, void **body_stream);
RB_API int rb_rebuild_cond_end(void *stream);

/* The gated rebuild in ONE launch: rb_bin + rb_nlist + rb_nlist_mirror
 * (same arguments and identical results) as phases of a single kernel
 * separated by grid-wide barriers; with rebuild_flag != NULL it exits at
 * once unless *rebuild_flag equals the step tag, so a captured step that
 * does not rebuild pays one launch instead of nine (or a conditional node).
 * `scratch` (rb_rebuild_scratch_bytes) must be zero-filled before its first
 * use (barrier words); every launch leaves it reusable. */
RB_API size_t rb_rebuild_scratch_bytes(int64_t n, int64_t ncell);
RB_API int rb_rebuild(const rb_grid *g, int64_t n, const double *pos, int32_t *cell_start,
                      int32_t *cell_particles, int32_t *cell_of_rank, double *pos_r,
                      int32_t *rank_of, double *x_ref, double r_list, int32_t capacity,
                      int32_t *rows, int32_t *row_count, int32_t *max_count, int32_t *mirror,
                      const int64_t *rebuild_flag, const unsigned long long *status, int64_t tag,
                      void *scratch, size_t scratch_bytes, void *stream);

/* Reusable captured step graphs (the domain loop's step kinds, recaptured
 * at every row rebuild): rb_graph_begin starts a thread-local capture on a
 * non-default stream; rb_graph_end ends it and instantiates into *exec, or,
 * when *exec already holds an executable, updates it in place
 * (cudaGraphExecUpdate; re-instantiates if the topology changed);
 * rb_graph_launch / rb_graph_destroy. */
RB_API int rb_graph_begin(void *stream);
RB_API int rb_graph_end(void *stream, uint64_t *exec);
RB_API int rb_graph_launch(uint64_t exec, void *stream);
RB_API int rb_graph_destroy(uint64_t exec);

/* One sample point of the device loop in a single launch: sums[0..4] =
 * (sum v^2 over the 3n velocity components, sum E2, W2, E3, W3 over the n
 * rank entries), each bit-identical to rb_reduce_sum(sq)_f64 of the same
 * array, and -- trace != NULL -- the rb_trace_record row.  `scratch`
 * (rb_sample_scratch_bytes) must be zero-filled before its first use; every
 * launch leaves it that way. */
RB_API size_t rb_sample_scratch_bytes(int64_t n);
RB_API int rb_sample(int64_t n, const double *vel, const double *e2_rank, const double *w2_rank,
                     const double *e3_rank, const double *w3_rank, double *sums,
                     const unsigned long long *status, int64_t sample_interval, double *trace,
                     void *scratch, size_t scratch_bytes, void *stream);

/* ---- device timing helpers for bench.py (events on the launch stream) -- */
/* FP64 FMA throughput microbenchmark: runs `iters` dependent-chain DFMA
 * blocks on every SM and returns the achieved FP64 TFLOP/s in *tflops. */
RB_API int rb_fp64_peak(int32_t iters, double *tflops, void *stream);
/* Writes `bytes` of a scratch buffer to evict L2 between timed steps. */
RB_API int rb_l2_flush(void *buf, size_t bytes, void *stream);
/* Timing events that can be recorded inside a CUDA-graph capture (external
 * event-record nodes): the bench brackets every step of a captured period
 * with them, so a step is timed from its first to its last kernel on the
 * device.  rb_event_elapsed returns milliseconds between two recorded
 * events (synchronises on the second). */
RB_API int rb_event_create(void **event);
RB_API int rb_event_destroy(void *event);
RB_API int rb_event_record(void *event, void *stream);
RB_API int rb_event_elapsed(void *start, void *end, float *ms);

#ifdef __cplusplus
}
#endif

#endif /* RESPA_B200_H */
