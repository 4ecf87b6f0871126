/*
 * oscb.h -- C ABI of the B200 oscillator Ising/Potts machine (liboscb.so).
 *
 * This is the drop-in boundary for the hot path of the reference package `oscim`
 * (paths below are relative to /root/reference/pkg/src/oscim/).  The reference has no FFI
 * layer of its own (it is numpy + numba); the seam it does have is the set of private kernel
 * signatures under its public solver API, and each entry point here replaces one of them:
 *
 *   oscb_graph_create_csr    CouplingMatrix CSR arrays handed to the kernels
 *                            (model.py:135-149, dynamics.py:250-251) and the canonical pair
 *                            list J.pairs() (model.py:238-242)
 *   oscb_graph_create_dense  the same couplings as a dense J (model.py:196-199), optionally one
 *                            row shard of it (multi-GPU dense path)
 *   oscb_initial_phases      NoiseSource.initial_phases             dynamics.py:127-129
 *   oscb_device_normals      NoiseSource.step_normals               dynamics.py:121-125
 *   oscb_step                trig precompute + _step_serial/_step_parallel, as called by
 *                            euler_step                             dynamics.py:155-190, 303-312
 *   oscb_score               _score_kernel                          dynamics.py:193-223
 *   oscb_energy              sample() energy                        dynamics.py:380
 *   oscb_run                 _simulate (time loop, noise, schedule, scoring cadence, best
 *                            tracking, traces, finite check)        dynamics.py:333-431
 *   oscb_dense_*             row-sharded dense step for one oversized graph
 *
 * Conventions: plain C types; all array arguments are caller-owned HOST buffers unless the
 * name says `_dev`; phases are float64 [R, n] row-major (replica-major) like the reference's
 * `phi`; every call returns 0 on success or one of the OSCB_E* codes, with a message in
 * oscb_last_error() (thread-local).  A handle owns one device, one CUDA stream and its
 * workspaces; calls on one handle must not overlap, different handles are independent.
 * There is no CPU fallback: without a usable CUDA device every call fails with OSCB_ECUDA.
 */
#ifndef OSCB_H_
#define OSCB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSCB_OK 0
#define OSCB_EINVAL 1    /* bad argument            -> ValueError     (dynamics.py:434-440) */
#define OSCB_ECUDA 2     /* CUDA / driver failure   -> RuntimeError                         */
#define OSCB_ENONFINITE 3 /* non-finite phase        -> NumericalError (dynamics.py:276-283) */
#define OSCB_ENOMEM 4

#define OSCB_OBJ_MAXCUT 0
#define OSCB_OBJ_COLORING 1

#define OSCB_PREC_F32 32 /* throughput mode: fp32 state and arithmetic                    */
#define OSCB_PREC_F64 64 /* parity mode: fp64, reference operation order                 */

#define OSCB_NOISE_DEVICE 0 /* counter-based Philox4x32-10 + Box-Muller, f(seed, step, i) */
#define OSCB_NOISE_HOST 1   /* caller supplies normals [steps, R, n] (parity hook)        */
#define OSCB_NOISE_NONE 2   /* kn treated as 0                                            */

#define OSCB_KERNEL_AUTO 0
#define OSCB_KERNEL_STREAM 1   /* one launch per step, phases in HBM/L2                   */
#define OSCB_KERNEL_RESIDENT 2 /* persistent CTA per replica tile, phases' (cos,sin) in smem */
#define OSCB_KERNEL_DENSE_TC 3 /* dense integer J: persistent tcgen05 int8 GEMM J*[cos|sin] digit planes */
#define OSCB_KERNEL_CLUSTER 4  /* latency mode: one replica per 8-CTA cluster, pairs exchanged through DSMEM */
#define OSCB_KERNEL_LOWDEG 5   /* low-degree graphs: persistent CTA per replica tile, phases in registers, pairs in smem */

typedef struct oscb_graph oscb_graph;

typedef struct oscb_graph_info {
    int64_t n;
    int64_t nnz;          /* directed nonzeros (2 per pair)                     */
    int64_t pairs;        /* canonical pairs i<j                                */
    int32_t device;
    int32_t is_dense;     /* 1 when created by oscb_graph_create_dense          */
    int32_t unit_weights; /* every stored coupling == 1.0                       */
    int32_t int_weights;  /* every stored coupling integer valued (exact scoring) */
    int64_t row_begin;    /* dense row shard [row_begin, row_end)               */
    int64_t row_end;
    int64_t max_degree;
} oscb_graph_info;

typedef struct oscb_run_params {
    double K, ks_max, ks_period, kn, h, t_stop; /* SolverParams fields (model.py:328-336)     */
    int32_t n_states;                           /* N                                          */
    int32_t objective;                          /* OSCB_OBJ_*                                 */
    int32_t precision;                          /* OSCB_PREC_*                                */
    int32_t noise_mode;                         /* OSCB_NOISE_*                               */
    int32_t kernel;                             /* OSCB_KERNEL_*                              */
    int32_t use_target;                         /* record first step reaching target_objective */
    int64_t steps;                              /* 0 => ceil(t_stop / h) (dynamics.py:349)    */
    int64_t cadence;                            /* 0 => reference rule (dynamics.py:325-330); <0 => never score between samples */
    double trace_stride;                        /* <= 0 => ks_period / 2 (dynamics.py:346)    */
    double target_objective;
    int64_t first_step;                         /* global index of the first step (restart)   */
    int32_t replicas_per_cta;                   /* 0 auto; resident kernel tile width         */
    int32_t variant;                            /* 0 auto; 1 = generic resident kernel even where the specialised float32 one applies;
                                                   dense tensor-core runs: 8 = stream J as int8, 4 = as packed e2m1 (the ranks of a
                                                   row-sharded run must all pass the same value -- connect checks it)            */
} oscb_run_params;

typedef struct oscb_run_outputs {
    /* any pointer may be NULL to skip that output */
    double *final_phases;    /* [R, n]                                                   */
    uint8_t *best_states;    /* [R, n]  state per oscillator of the best-scored sample   */
    double *best_objective;  /* [R]     objective of best_states (dynamics.py:421)       */
    double *trace_t;         /* [max_samples]                                            */
    double *trace_ks;        /* [max_samples]                                            */
    double *energy;          /* [R, max_samples]  (dynamics.py:380)                      */
    double *best_trace;      /* [R, max_samples]  best-so-far at each sample             */
    int64_t *first_hit_step; /* [R] first scored step with objective >= / <= target, -1 if never */
    int64_t max_samples;
    /* filled by the call */
    int64_t n_samples;
    int64_t steps_executed;
    int64_t nonfinite[3];    /* {replica row, oscillator, step} when OSCB_ENONFINITE     */
    double device_ms;        /* CUDA-event time of the integrate loop only               */
    int64_t kernel_launches; /* kernels launched inside that region                      */
    int32_t kernel_used;     /* OSCB_KERNEL_*                                            */
    int32_t replicas_per_cta;
    int64_t smem_bytes;
} oscb_run_outputs;

const char *oscb_last_error(void);
int oscb_version(void);
int oscb_device_count(int *count);
/* Device workspaces are recycled through a size-keyed pool between calls; this frees the parked
 * blocks (cudaFree).  Never needed for correctness. */
int oscb_pool_trim(void);

/* Symmetric CSR from an edge list, built on the device: the GPU form of CouplingMatrix.from_edges (reference
 * model.py:151-200).  m entries (i[e], j[e], x[e]), one per unordered pair, HOST buffers; out: indptr [n + 1], indices and data
 * [*nnz <= 2 m] (caller provides 2 m entries each), rows and the columns of a row ascending, entries with x == 0 dropped -- bit
 * for bit what the reference's host build returns.  OSCB_EINVAL with the reference's messages, in the reference's order: an
 * index outside [0, n), a diagonal entry, a pair listed twice (zero-valued entries count).  device_ms (may be NULL): time of
 * the kernels alone, CUDA events.  n < 2^31. */
int oscb_csr_from_edges(int device, int64_t n, int64_t m, const int64_t *i, const int64_t *j, const double *x,
                        int64_t *indptr, int64_t *indices, double *data, int64_t *nnz, double *device_ms);
int oscb_graph_create_csr(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                          const double *data, oscb_graph **out);
/* Dense couplings.  Integer couplings |J| <= 127 on 128-row aligned shards also get the tile images of the
 * tensor-core kernel (OSCB_KERNEL_DENSE_TC), whose sums are exact integers while the accumulators hold them: the
 * int8 stream needs max_i sum_j |J_ij| * 128 < 2^31, the packed e2m1 stream (every coupling in {0, +-1, +-2, +-3,
 * +-4, +-6}) max_i sum_j |J_ij| * 4 < 2^24.  A graph that breaks a bound is kept off that stream (it then runs on
 * the SIMT dense kernels), never rounded silently. */
int oscb_graph_create_dense(int device, int64_t n, const double *J, int64_t row_begin,
                            int64_t row_end, oscb_graph **out);
int oscb_graph_destroy(oscb_graph *g);
int oscb_graph_get_info(const oscb_graph *g, oscb_graph_info *info);

int oscb_initial_phases(oscb_graph *g, const uint64_t *seeds, int64_t R, double *phi_out);

/* The device noise source (replaces NoiseSource.step_normals, dynamics.py:121-125): the standard
 * normals the integrator draws for `seed` at `step`, oscillators 0..n-1, in the arithmetic of
 * `precision`, widened to float64.  A pure function of (seed, step, oscillator). */
int oscb_device_normals(int device, uint64_t seed, int64_t step, int64_t n, int32_t precision,
                        double *out /* [n] */);

int oscb_step(oscb_graph *g, int64_t R, const double *phi_in, const double *noise, double K,
              double ks, double h, double kn_sqrt_h, int32_t n_states, int32_t precision,
              double *phi_out, int64_t *nonfinite /* [2] replica, oscillator; -1 if none */);

int oscb_score(oscb_graph *g, int64_t R, const double *phi, int32_t n_states, int32_t maximize,
               int64_t *states /* [R, n] or NULL */, double *objective /* [R] */);

int oscb_energy(oscb_graph *g, int64_t R, const double *phi, double *energy /* [R] */);

int oscb_run(oscb_graph *g, const oscb_run_params *params, const uint64_t *seeds, int64_t R,
             const double *phi0 /* [R, n] or NULL => Philox initial phases */,
             const double *noise /* [steps, R, n] when noise_mode == OSCB_NOISE_HOST */,
             oscb_run_outputs *out);

/* ---- one oversized dense graph, row-sharded over several GPUs ------------------
 * Every rank creates its shard with oscb_graph_create_dense(device, n, J_rows, row_begin, row_end)
 * and owns the phases of those rows.  Per Euler step each rank calls oscb_dense_shard_step on the
 * FULL phase array (all n oscillators, device memory, layout [n][R] replica-minor, float32 or
 * float64 by `precision`) and gets the new phases of ITS rows ([rows][R]); the host side then
 * all-gathers the slices (NCCL through torch.distributed) into the next full array.  These calls
 * take DEVICE pointers and enqueue on `stream` (a cudaStream_t; NULL = the handle's own stream)
 * without synchronising, so they compose with the collective on the same stream.
 *   oscb_dense_shard_step       trig precompute + _step_* for the shard's rows  dynamics.py:393-401
 *   oscb_dense_shard_objective  this shard's part of _score_kernel's sum        dynamics.py:214-223
 *                               (sum over ranks = the objective; all-reduce it)
 *   oscb_dense_shard_energy     this shard's part of the sample() energy        dynamics.py:380
 *   oscb_graph_nonfinite        first non-finite (replica, oscillator, step) seen by the handle */
typedef struct oscb_shard_step_params {
    double K, ks, h, kn_sqrt_h;
    int32_t n_states, precision, noise_on, reserved;
    int64_t step;                       /* global step index (noise counter, non-finite report) */
} oscb_shard_step_params;

int oscb_dense_shard_step(oscb_graph *g, int64_t R, const oscb_shard_step_params *p,
                          const void *phi_full_dev, void *phi_rows_out_dev,
                          const uint64_t *seeds_dev /* [R] */, void *stream);
int oscb_dense_shard_objective(oscb_graph *g, int64_t R, int32_t precision, const void *phi_full_dev,
                               int32_t n_states, int32_t maximize, double *partial_dev /* [R] */,
                               void *stream);
int oscb_dense_shard_energy(oscb_graph *g, int64_t R, int32_t precision, const void *phi_full_dev,
                            double *partial_dev /* [R] */, void *stream);
int oscb_graph_nonfinite(oscb_graph *g, int64_t where[3] /* replica, oscillator, step; -1 if none */,
                         int32_t reset);

/* ---- the same row-sharded dense run FUSED: one persistent tensor-core kernel per rank ---------
 * (csrc/oscb_umma.cuh).  J (integer couplings |J| <= 127, shards aligned to 128 rows) is streamed
 * as int8 tile images through tcgen05.mma against the int8 digit planes of (cos, sin); the epilogue
 * of every Euler step writes the new digits of the rank's rows straight into EVERY rank's next-step
 * image (peer memory over NVLink: the per-step all-gather of oscb_dense_shard_step + NCCL becomes
 * stores from inside the kernel), adds its part of the cut into every rank's event record
 * (system-scope atomics) and arrives on every rank's step counter.  No host code runs between
 * steps.  Replaces, per rank: trig precompute + _step_* + _score_kernel + sample() of
 * dynamics.py:387-410 for the rank's rows, and the phase exchange between them.
 *
 *   create   : schedule (steps, sample steps, scoring cadence from `pair_count` of the WHOLE graph
 *              when params->cadence == 0) and buffers for R <= 28 replicas
 *   export   : OSCB_FUSED_MEM_BYTES describing this rank's exchange block (CUDA IPC handle +
 *              address + grid size); all-gather these blobs over the ranks (any host transport)
 *   connect  : map every peer's block (cudaIpcOpenMemHandle; plain addresses inside one process)
 *   prepare  : zero the block, build the pass-0 state from phi0 ([R, n] of the WHOLE graph, or
 *              NULL for the Philox initial phases).  Host-barrier over the ranks after this call.
 *   launch   : enqueue the kernel (asynchronous)
 *   finish   : wait; outputs as oscb_run, except final_phases / best_states hold THIS RANK's rows
 *              only ([R, rows], rows from oscb_dense_fused_rows); objectives, traces and energies
 *              are complete on every rank. */
typedef struct oscb_fused oscb_fused;
#define OSCB_FUSED_MEM_BYTES 96
int oscb_dense_fused_create(oscb_graph *shard, const oscb_run_params *params, int64_t R, int64_t pair_count,
                            int32_t world, int32_t rank, oscb_fused **out);
int oscb_dense_fused_export(oscb_fused *f, void *mem /* [OSCB_FUSED_MEM_BYTES] */);
int oscb_dense_fused_connect(oscb_fused *f, const void *all /* [world * OSCB_FUSED_MEM_BYTES], rank order */);
int oscb_dense_fused_prepare(oscb_fused *f, const uint64_t *seeds /* [R] */, const double *phi0 /* [R, n] or NULL */);
int oscb_dense_fused_launch(oscb_fused *f);
int oscb_dense_fused_finish(oscb_fused *f, oscb_run_outputs *out);
/* CTAs this rank's persistent kernel launches and how many of them share one 128-row tile of J (split-K: a rank that
 * owns few row tiles splits each tile's K range over SMs / tiles CTAs; the partial sums meet in a global int32
 * accumulator, so the results do not depend on it). */
int oscb_dense_fused_grid(const oscb_fused *f, int32_t *ctas, int32_t *splits);
int oscb_dense_fused_rows(const oscb_fused *f, int64_t *rows);
int oscb_dense_fused_destroy(oscb_fused *f);
/* What a tensor-core dense run of R replicas on this handle streams: bits per coupling of the J
 * image it reads every Euler step (8 = int8 tiles; 4 = packed e2m1 tiles, taken when every coupling
 * is in {0, +-1, +-2, +-3, +-4, +-6} and the R replicas fit one launch of that stream: 12 at N = 2) and the replicas one
 * launch integrates (R above that runs as several launches).  OSCB_EINVAL when the handle has no
 * tensor-core plan (non-integer couplings, or not a dense handle). */
int oscb_dense_tc_stream(const oscb_graph *g, int32_t n_states, int64_t R, int32_t *coupling_bits,
                         int32_t *replicas_per_launch);

/* Device self-test behind the scoring shortcuts of the float32 kernel: counts the float32 phases in
 * [0, 1) (all 2^30-ish of them) whose sign-bit-of-cosine state (N = 2), or whose state from the
 * float32 decision-boundary table (N = 3..8), differs from the reference threshold
 * (dynamics.py:203-213); also bounds the error of the fast trig.  Must return 0 mismatches. */
int oscb_selftest_sign_state(int device, uint64_t *mismatches);

/* Host-only: the stream compiler of the low-degree persistent kernel (OSCB_KERNEL_LOWDEG; no GPU needed).  For a
 * tile of `replicas_per_cta` replicas (a power of two <= 32), `warps` warps per CTA and `items_per_thread` quads
 * per thread it returns the position -> quad map quad_of [warps * items_per_thread * C] (C = 32 / replicas_per_cta;
 * >= ceil(n / 4): no quad), the component-major slot of every oscillator slot_of [n], and the ELL stream of
 * 4-neighbour groups: offsets [4 * entries] (slot * replicas_per_cta * 8 bytes; bit 31 of a group's 4th offset marks
 * the last group of a row when the graph is not uniform, i.e. has a row of more than 4 neighbours) and couplings
 * [4 * entries] (padding: an all-zero pad slot, coupling 0).  Call once with NULL buffers for
 * `entries`.  Restates the traversal of the CSR rows of dynamics.py:166-170 for that kernel. */
int oscb_lowdeg_plan_host(int64_t n, const int64_t *indptr, const int64_t *indices, const double *weights,
                          int32_t replicas_per_cta, int32_t warps, int32_t items_per_thread, int32_t *uniform,
                          int64_t *group_rows, int64_t *entries, uint32_t *quad_of, uint32_t *slot_of,
                          uint32_t *offsets, float *couplings, int32_t *warp_start);

/* The same for k_lowdeg_pair, the two-replicas-per-lane form (N = 2 max-cut rows of any degree; C = 64 / replicas_per_cta
 * slots per warp, replicas_per_cta >= 2).  On a looped stream the four rows of a quad are visited in descending degree:
 * bits 24..31 of a quad_of word hold the component (0..3) visited 1st..4th, two bits each, bits 0..23 the quad (all ones:
 * none), and slot_of is (visiting position) * Qp + position of the quad.  A row's neighbours -- and its padding, which may
 * sit anywhere in the row -- are ordered so that the slots read by one quarter-warp fall in different shared-memory bank
 * groups where the row contents allow it. */
int oscb_lowdeg_pair_plan_host(int64_t n, const int64_t *indptr, const int64_t *indices, const double *weights,
                               int32_t replicas_per_cta, int32_t warps, int32_t items_per_thread, int32_t *uniform,
                               int64_t *group_rows, int64_t *entries, uint32_t *quad_of, uint32_t *slot_of,
                               uint32_t *offsets, float *couplings, int32_t *warp_start);

/* Host-only: the graph compiler of the persistent kernel (no GPU needed).  Turns a canonical CSR
 * (model.py:135-149) into the sliced-ELL neighbour stream for tiles of `replicas_per_cta`
 * replicas, CTAs of at most `max_threads` threads and (cos, sin) pairs of `pair_bytes` bytes.
 * keep_order != 0 keeps every row in CSR order (float64 parity mode).  Call once with
 * ids == NULL for the sizes, then with buffers: warp_start [warps], rows [warps*rounds*4*C],
 * ginfo [warps*rounds], ids [4*(group_rows+1)*C] with C = 32/(replicas_per_cta/replicas_per_lane)
 * slots per warp (a lane of the float32 kernel may own 2 adjacent replicas).  Row and
 * neighbour ids are pre-multiplied by replicas_per_cta; values >= n*replicas_per_cta are padding. */
int oscb_resident_plan_host(int64_t n, const int64_t *indptr, const int64_t *indices,
                            int32_t replicas_per_cta, int32_t replicas_per_lane, int32_t max_threads, int32_t pair_bytes,
                            int32_t keep_order, int32_t *warps, int32_t *rounds, int64_t *group_rows,
                            int64_t *bank_conflicts, int32_t *warp_start, uint16_t *rows,
                            uint32_t *ginfo, uint16_t *ids);

#ifdef __cplusplus
}
#endif
#endif /* OSCB_H_ */
