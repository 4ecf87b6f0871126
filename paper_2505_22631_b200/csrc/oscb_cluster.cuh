// oscb_cluster.cuh -- latency mode of the float32 integrator: ONE replica spread over a thread-block
// cluster of 8 or 16 SMs (the reference's default `solve` is a single replica, cli.py:143-153; at
// R = 1 the persistent kernel of oscb_resident_fast.cuh keeps a whole run on one SM).
//
//   * every CTA of the cluster holds a full copy of the (cos, sin) pairs of all n oscillators in
//     shared memory, double buffered, and owns n / CL rows of J (CL = cluster size) (their CSR slice sits in its
//     shared memory too);
//   * phase A of a step: a row is gathered by 8 lanes (neighbours strided over the lanes, 3 shuffle
//     stages); phase B: one thread per row does the Euler update (SHIL, noise, wrap;
//     dynamics.py:166-172) and stores the new pair straight into the NEXT buffer of all CL CTAs
//     through distributed shared memory, while the remaining warps draw the next step's Philox
//     noise (it does not depend on the sums, so it stays off the critical path);
//   * one cluster barrier (arrive.release / wait.acquire) ends the step; nothing leaves the SMs.
//   * N = 2 max-cut scoring rides on the next step's gather (sign bit of the gathered cosine = the
//     neighbour's lattice state, see oscb_resident_fast.cuh); the per-CTA partial cuts are
//     exchanged through DSMEM on the same barrier, and every CTA keeps the same best-so-far.
//
// Same arithmetic as k_resident_fast (float32, trig_turns_direct, normals4_fast, the same
// (seed, step, oscillator) noise); the summation order over a row differs, so the two agree to
// rounding, like any two float32 tile shapes.
#pragma once
#include "oscb_resident_fast.cuh"
#include <cooperative_groups.h>

namespace oscb {

namespace cg = cooperative_groups;

constexpr int CL_MAX = 16;    // CTAs per cluster: 8 (portable maximum) or 16 (non-portable size, taken while 16 SMs per replica are free)
constexpr int CL_LPR = 8;    // lanes per row

struct ClusterArgs {
    int n, n_al, rows_per_cta, nnz_cap, weighted, R_real;
    int noise_on, use_target, initial_sample, n_sample_steps, sample_offset;
    float hK, knsh;
    long long step_begin, step_end, cadence, trace_stride;
    double target;
    uint32_t off_cs, off_phi, off_st, off_rowptr, off_rowsum, off_sums, off_negw, off_kick, off_col, off_w, off_xpart, off_red, off_misc, smem_total;
    const int *indptr, *indices;
    const float *w32;
    const float *hks_table;
    double *phi_io;                    // [R][n] float64, host layout: initial phases in, final phases out
    const uint64_t *seeds;
    const long long *sample_steps;
    double *best_obj, *energy, *best_trace;
    uint8_t *best_states;              // [R][n]
    long long *first_hit;
    unsigned long long *nonfinite;
    long long *dbg;                    // optional [4]: cycles of CTA 0 in phase A / phase B / cluster barrier / rest
};

struct ClusterSmem {
    size_t cs, phi, st, rowptr, rowsum, sums, negw, kick, col, w, xpart, red, misc, total;
    __host__ static ClusterSmem make(int n_al, int rows_per_cta, int nnz_cap, bool weighted)
    {
        ClusterSmem s;
        size_t o = 0;
        auto take = [&](size_t bytes) { size_t at = o; o += (bytes + 15) & ~(size_t)15; return at; };
        s.cs = take((size_t)2 * n_al * 8);
        s.phi = take((size_t)rows_per_cta * 4);
        s.st = take((size_t)rows_per_cta);
        s.rowptr = take((size_t)(rows_per_cta + 1) * 4);
        s.rowsum = take((size_t)rows_per_cta * 4);
        s.sums = take((size_t)rows_per_cta * 8);
        s.negw = take((size_t)rows_per_cta * 4);
        s.kick = take((size_t)2 * 4 * ((rows_per_cta + 3) / 4) * 4);
        s.col = take((size_t)nnz_cap * 2);
        s.w = take(weighted ? (size_t)nnz_cap * 4 : 0);
        s.xpart = take((size_t)4 * 2 * CL_MAX * 8);
        s.red = take((size_t)32 * 2 * 8);
        s.misc = take(64);
        s.total = o;
        return s;
    }
};

template <int CL_SIZE>
__global__ void __cluster_dims__(CL_SIZE, 1, 1) __launch_bounds__(1024, 1) k_cluster_fast(const ClusterArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int replica = blockIdx.x / CL_SIZE;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
    const int sub = tid & (CL_LPR - 1), group = tid / CL_LPR, groups = NT / CL_LPR;
    const int rounds = (a.rows_per_cta + groups - 1) / groups;
    const bool live = replica < a.R_real;

    float2 *cs = reinterpret_cast<float2 *>(smem_raw + a.off_cs);            // [2][n_al]
    float *phi_s = reinterpret_cast<float *>(smem_raw + a.off_phi);
    uint8_t *st_s = smem_raw + a.off_st;
    int *rowptr_s = reinterpret_cast<int *>(smem_raw + a.off_rowptr);
    float *rowsum_s = reinterpret_cast<float *>(smem_raw + a.off_rowsum);
    float2 *sums_s = reinterpret_cast<float2 *>(smem_raw + a.off_sums);
    float *negw_s = reinterpret_cast<float *>(smem_raw + a.off_negw);
    float *kick_s = reinterpret_cast<float *>(smem_raw + a.off_kick);          // [2][4 * quads]
    uint16_t *col_s = reinterpret_cast<uint16_t *>(smem_raw + a.off_col);
    float *w_s = reinterpret_cast<float *>(smem_raw + a.off_w);
    double *xpart = reinterpret_cast<double *>(smem_raw + a.off_xpart);      // [4 slots][2: objective, energy][CL_SIZE]
    double *red = reinterpret_cast<double *>(smem_raw + a.off_red);          // [32][2]
    double *best_s = reinterpret_cast<double *>(smem_raw + a.off_misc);
    int *improved_s = reinterpret_cast<int *>(smem_raw + a.off_misc + 8);

    const int row0 = rank * a.rows_per_cta;
    const int my_rows = max(0, min(a.n, row0 + a.rows_per_cta) - row0);
    const uint64_t seed = a.seeds[live ? replica : 0];
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));

    // ---- prologue: this CTA's CSR slice, the pairs of ALL oscillators, the phases of its own rows ----
    {
        const int e0 = my_rows > 0 ? a.indptr[row0] : 0;
        for (int r = tid; r <= my_rows; r += NT) rowptr_s[r] = a.indptr[row0 + r] - e0;
        const int cnt = my_rows > 0 ? a.indptr[row0 + my_rows] - e0 : 0;
        for (int e = tid; e < cnt; e += NT) {
            col_s[e] = (uint16_t)a.indices[e0 + e];
            if (a.weighted) w_s[e] = a.w32[e0 + e];
        }
        const double *src = a.phi_io + (size_t)(live ? replica : 0) * a.n;
        for (int i = tid; i < a.n_al; i += NT) {
            float s = 0.f, c = 0.f;
            if (i < a.n) trig_turns_direct((float)src[i], s, c);
            cs[i] = make_float2(c, s);
            cs[a.n_al + i] = make_float2(0.f, 0.f);
        }
        for (int r = tid; r < my_rows; r += NT) phi_s[r] = (float)src[row0 + r];
        if (tid == 0) { *best_s = a.best_obj[live ? replica : 0]; *improved_s = 0; }
        __syncthreads();
        for (int r = tid; r < my_rows; r += NT) {
            float t = 0.f;
            if (a.weighted)
                for (int e = rowptr_s[r]; e < rowptr_s[r + 1]; ++e) t += w_s[e];
            rowsum_s[r] = t;
        }
    }
    cluster.sync();

    int xslot = 0;   // exchange slot counter, advances identically in every CTA

    // CTA-wide sum of (x, y) in a fixed order; result valid in thread 0
    auto block_sum2 = [&](double x, double y, double &ox, double &oy) {
        for (int off = 16; off > 0; off >>= 1) {
            x += __shfl_down_sync(0xffffffffu, x, off);
            y += __shfl_down_sync(0xffffffffu, y, off);
        }
        if (lane == 0) { red[2 * warp] = x; red[2 * warp + 1] = y; }
        __syncthreads();
        ox = 0.0; oy = 0.0;
        if (tid == 0)
            for (int w = 0; w < nwarps; ++w) { ox += red[2 * w]; oy += red[2 * w + 1]; }
        __syncthreads();
    };
    // thread 0's CTA partial -> slot `xslot` of every CTA of the cluster (DSMEM)
    auto publish_partial = [&](double obj2, double en2) {
        if (tid == 0) { red[0] = obj2; red[1] = en2; }
        __syncthreads();
        if (tid < CL_SIZE) {
            double *remote = cluster.map_shared_rank(xpart, tid);
            remote[(xslot * 2 + 0) * CL_SIZE + rank] = red[0];
            remote[(xslot * 2 + 1) * CL_SIZE + rank] = red[1];
        }
    };
    // after the barrier: totals of slot `xslot` (same order in every CTA), best-so-far, states
    auto settle = [&](long long label, int sample_col) {
        if (tid == 0) {
            double obj2 = 0.0, en2 = 0.0;
            for (int r = 0; r < CL_SIZE; ++r) { obj2 += xpart[(xslot * 2 + 0) * CL_SIZE + r]; en2 += xpart[(xslot * 2 + 1) * CL_SIZE + r]; }
            const double obj = 0.5 * obj2;
            const bool better = obj > *best_s;
            *improved_s = better ? 1 : 0;
            if (better) {
                *best_s = obj;
                if (rank == 0 && live && a.use_target && a.first_hit[replica] < 0 && obj >= a.target) a.first_hit[replica] = label;
            }
            if (sample_col >= 0 && rank == 0 && live) {
                a.energy[(size_t)replica * a.trace_stride + sample_col] = 0.5 * en2;
                a.best_trace[(size_t)replica * a.trace_stride + sample_col] = *best_s;
            }
        }
        __syncthreads();
        if (*improved_s && live)
            for (int r = tid; r < my_rows; r += NT) a.best_states[(size_t)replica * a.n + row0 + r] = st_s[r];
        xslot = (xslot + 1) & 3;
        __syncthreads();
    };
    // explicit scoring of the pairs in buffer `buf` (trace samples, the first and the last state)
    auto score_explicit = [&](int buf, long long label, int sample_col) {
        const float2 *cur = cs + (size_t)buf * a.n_al;
        double obj2 = 0.0, en2 = 0.0;
        for (int k = 0; k < rounds; ++k) {
            const int rl = group + k * groups;
            const bool valid = rl < my_rows;
            const int beg = valid ? rowptr_s[rl] : 0, end = valid ? rowptr_s[rl + 1] : 0;
            const float2 own = valid ? cur[row0 + rl] : make_float2(0.f, 0.f);
            const bool own1 = __float_as_int(own.x) < 0;
            double cutw = 0.0, en = 0.0;
            for (int e = beg + sub; e < end; e += CL_LPR) {
                const float2 v = cur[col_s[e]];
                const double w = a.weighted ? (double)w_s[e] : 1.0;
                if ((__float_as_int(v.x) < 0) != own1) cutw += w;
                en += w * ((double)own.x * (double)v.x + (double)own.y * (double)v.y);
            }
            for (int off = CL_LPR / 2; off > 0; off >>= 1) {
                cutw += __shfl_xor_sync(0xffffffffu, cutw, off);
                en += __shfl_xor_sync(0xffffffffu, en, off);
            }
            if (sub == 0 && valid) { obj2 += cutw; en2 += en; st_s[rl] = own1 ? 1 : 0; }
        }
        double o, e;
        block_sum2(obj2, en2, o, e);
        publish_partial(o, e);
        cluster.sync();
        settle(label, sample_col);
    };

    int sample_cur = 0;
    while (sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] < a.step_begin) ++sample_cur;
    if (a.initial_sample) score_explicit(0, -1, 0);

    bool pending = false;
    long long pending_label = 0;
    long long next_sample_step = sample_cur < a.n_sample_steps ? a.sample_steps[sample_cur] : -1;
    // steps until the next multiple of the cadence (no 64-bit division inside a 2 us step)
    long long cad_left = a.cadence > 0 ? (a.cadence - a.step_begin % a.cadence) % a.cadence : -1;
    long long dbg_acc[3] = {0, 0, 0};
    const long long dbg_t0 = a.dbg ? clock64() : 0;

    // Work split of a step.  Phase A (all warps): 8 lanes gather one row.  Phase B: one thread per row (the
    // first WB warps) does the Euler update and publishes the new pair to the 8 CTAs, while the other warps
    // draw the NEXT step's noise (one thread per quad of rows, one Philox block each) -- the draw does not
    // depend on the sums, so it never sits on the critical path.
    const int WB = max(1, min(nwarps - 1, (a.rows_per_cta + 31) / 32));
    const int quads = (a.rows_per_cta + 3) / 4;
    auto draw_noise_for = [&](long long step_of, float *dst) {          // called by the threads of warps >= WB
        const int nt = (nwarps - WB) * 32;
        for (int q = tid - WB * 32; q < quads; q += nt) {
            const int i0 = row0 + 4 * q;
            float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
            if (a.noise_on && i0 < a.n)
                normals4_fast(philox4x32_10(make_uint4((uint32_t)i0 >> 2, (uint32_t)step_of, (uint32_t)(step_of >> 32), 0x6F736362u), key),
                              z0, z1, z2, z3);
            dst[4 * q + 0] = z0; dst[4 * q + 1] = z1; dst[4 * q + 2] = z2; dst[4 * q + 3] = z3;
        }
    };
    if (warp >= WB) draw_noise_for(a.step_begin, kick_s);
    __syncthreads();

#pragma unroll 1
    for (long long step = a.step_begin; step < a.step_end; ++step) {
        const int cur_i = (int)((step - a.step_begin) & 1);
        const float2 *cur = cs + (size_t)cur_i * a.n_al;
        float2 *nxt = cs + (size_t)(cur_i ^ 1) * a.n_al;
        const float *kick_cur = kick_s + (size_t)cur_i * 4 * quads;
        float *kick_nxt = kick_s + (size_t)(cur_i ^ 1) * 4 * quads;
        const float hks = __ldg(a.hks_table + (step - a.step_begin));
        const bool is_sample = step == next_sample_step;
        const bool cadence_hit = cad_left == 0;
        if (a.cadence > 0) cad_left = cad_left == 0 ? a.cadence - 1 : cad_left - 1;
        const bool count_now = pending;

        long long c0 = 0, c1 = 0, c2 = 0, c3 = 0;
        if (a.dbg) c0 = clock64();
        // ---- phase A: row sums.  64 neighbours of a row at a time: 8 per lane, all index loads first, then all
        // pair loads (independent: one shared-memory latency, not eight), then the adds ----
        for (int k = 0; k < rounds; ++k) {
            const int rl = group + k * groups;
            const bool valid = rl < my_rows;
            const int beg = valid ? rowptr_s[rl] : 0, end = valid ? rowptr_s[rl + 1] : 0;
            float2 sum = make_float2(0.f, 0.f);
            float negw = 0.f;
            for (int e0 = beg + sub; e0 < end; e0 += 8 * CL_LPR) {
                int col[8];
                float wt[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int e = e0 + u * CL_LPR;
                    const bool ok = e < end;
                    col[u] = ok ? (int)col_s[e] : a.n;                  // pair n of every buffer is (0, 0)
                    wt[u] = (ok && a.weighted) ? w_s[e] : 1.f;
                }
                float2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = cur[col[u]];
                if (a.weighted) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) sum = __ffma2_rn(make_float2(wt[u], wt[u]), v[u], sum);
                } else {
                    sum = __fadd2_rn(sum, __fadd2_rn(__fadd2_rn(__fadd2_rn(v[0], v[1]), __fadd2_rn(v[2], v[3])),
                                                     __fadd2_rn(__fadd2_rn(v[4], v[5]), __fadd2_rn(v[6], v[7]))));
                }
                if (count_now) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) negw += __float_as_int(v[u].x) < 0 ? wt[u] : 0.f;   // unit weights: a count, exact in float32
                }
            }
            for (int off = CL_LPR / 2; off > 0; off >>= 1) {
                sum.x += __shfl_xor_sync(0xffffffffu, sum.x, off);
                sum.y += __shfl_xor_sync(0xffffffffu, sum.y, off);
            }
            if (count_now)
                for (int off = CL_LPR / 2; off > 0; off >>= 1) negw += __shfl_xor_sync(0xffffffffu, negw, off);
            if (sub == 0 && valid) {
                sums_s[rl] = sum;
                if (count_now) negw_s[rl] = negw;
            }
        }
        __syncthreads();
        if (a.dbg) c1 = clock64();

        // ---- phase B: update + publish (warps < WB), next step's noise (the others) ----
        double twice_cut = 0.0;
        if (warp < WB) {
            for (int rl = tid; rl < my_rows; rl += WB * 32) {
                const int i = row0 + rl;
                const float2 own = cur[i], sum = sums_s[rl];
                const float ci = own.x, si = own.y, p = phi_s[rl];
                if (count_now) {
                    const bool own1 = __float_as_int(ci) < 0;
                    st_s[rl] = own1 ? 1 : 0;
                    const float all = a.weighted ? rowsum_s[rl] : (float)(rowptr_s[rl + 1] - rowptr_s[rl]);
                    twice_cut += (double)(own1 ? all - negw_s[rl] : negw_s[rl]);
                }
                const float acc = si * sum.x - ci * sum.y;
                const float x = fmaf(a.hK, acc, fmaf(-hks, si * ci, fmaf(a.knsh, kick_cur[rl], p)));
                const float w = x - floorf(x);
                const float y = (w >= 1.0f) ? 0.0f : w;
                if (!(fabsf(x) < INFINITY) && live) flag_nonfinite(a.nonfinite, (uint64_t)step, (uint32_t)replica, (uint32_t)i);
                phi_s[rl] = y;
                float s2, c2;
                trig_turns_direct(y, s2, c2);
                const float2 np = make_float2(c2, s2);
#pragma unroll
                for (int r = 0; r < CL_SIZE; ++r) cluster.map_shared_rank(nxt, r)[i] = np;   // DSMEM: the next buffer of every CTA
            }
        } else if (step + 1 < a.step_end) {
            draw_noise_for(step + 1, kick_nxt);
        }
        if (count_now) {
            double o, e;
            block_sum2(twice_cut, 0.0, o, e);
            publish_partial(o, 0.0);
        }
        if (a.dbg) c2 = clock64();
        cluster.sync();            // every CTA's new pairs (and partial cuts) have landed everywhere
        if (a.dbg) c3 = clock64();
        if (a.dbg && tid == 0 && blockIdx.x == 0) { dbg_acc[0] += c1 - c0; dbg_acc[1] += c2 - c1; dbg_acc[2] += c3 - c2; }
        if (count_now) {
            settle(pending_label, -1);
            pending = false;
        }
        if (is_sample) {
            score_explicit(cur_i ^ 1, step, a.sample_offset + sample_cur);
            ++sample_cur;
            next_sample_step = sample_cur < a.n_sample_steps ? a.sample_steps[sample_cur] : -1;
        } else if (cadence_hit) {
            if (step + 1 < a.step_end) { pending = true; pending_label = step; }
            else score_explicit(cur_i ^ 1, step, -1);
        }
    }
    if (a.dbg && tid == 0 && blockIdx.x == 0) { a.dbg[0] = dbg_acc[0]; a.dbg[1] = dbg_acc[1]; a.dbg[2] = dbg_acc[2]; a.dbg[3] = clock64() - dbg_t0; }
    if (tid == 0 && rank == 0 && live) a.best_obj[replica] = *best_s;
    if (live)
        for (int r = tid; r < my_rows; r += NT) a.phi_io[(size_t)replica * a.n + row0 + r] = (double)phi_s[r];
    cluster.sync();                // no CTA exits while a peer may still address its shared memory
}

} // namespace oscb
