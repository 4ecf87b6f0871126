// oscb_lowdeg.cuh -- the persistent float32 Euler kernel for LOW-DEGREE graphs (toroidal GSET shapes such
// as G81, SATLIB flat* colouring instances: a handful of neighbours per oscillator).
//
// At degree 4 a row's gather is a dozen instructions and the per-oscillator work (noise, trig, update,
// read-out) is everything; k_resident_fast's sliced-ELL machinery (row tables, group counts, 16-bit row ids,
// phases in L2, staged pairs) then costs more than the arithmetic.  This kernel keeps the same dynamics,
// noise stream, read-out rule and result contract (dynamics.py:155-223, :333-431) and strips the rest:
//
//   * a thread OWNS its work items for the whole run.  An item is one quad (4 consecutive oscillators = one
//     Philox block) of one replica; its four PHASES LIVE IN REGISTERS (QPT items per thread, a template
//     parameter, fully unrolled) -- no phase traffic at all, the first load and the last store aside;
//   * shared memory holds only the (cos, sin) pairs, in component-major order: slot(i) = (i & 3) * Qp +
//     position(i >> 2), so the 32 / RT quads a warp-instruction touches sit next to each other -- own loads,
//     own stores and, on lattice-like graphs, the neighbour gathers are conflict-free;
//   * a step is pass A (gather + update into the registers) | barrier | pass B (trig of the new phase, the
//     pair stored to its slot) | barrier.  Nothing is staged through L2;
//   * the neighbour stream is ELL with 4-neighbour groups, read straight from global memory (L2) by the lane
//     that uses it, coalesced: {4 x u16 slot ids, 4 x f16 couplings} = 16 B per group for N = 2 (integer
//     couplings are exact in f16; unit weights are the same stream with 1.0), 8 B for the unit-weight
//     N = 3 colouring.  UNIFORM graphs (every row <= 4 neighbours) have exactly one group per row at an
//     address known at compile time up to a stride -- straight-line code; otherwise a warp walks its
//     groups with a running pointer and a "last group of the row" flag in the stream itself;
//   * read-out rides on the gather of the NEXT step (as in k_resident_fast): for N = 2 the sign bit of a stored
//     cosine is the oscillator's lattice state, and cut = (W - sum_i sigma_i sum_j w_ij sigma_j) / 4 needs one
//     LOP3 + one FADD per neighbour; for N = 3 the low three mantissa bits of the stored cosine hold the
//     state one-hot (a <= 7 ulp perturbation of a value whose own MUFU error is larger), so the count of
//     equal-state neighbours is one AND + one add per neighbour.  Trace samples ride the same way, the
//     energy being sum_i (c_i, s_i) . sum_j w_ij (c_j, s_j) / 2 of the gather sums that are there anyway.
//
// Arithmetic of a step (float32, FMA-contracted) is k_resident_fast's; parity is by tolerance and distribution.
#pragma once
#include "oscb_resident_fast.cuh"
#include <cuda_fp16.h>

namespace oscb {

#define OSCB_LD_PADS 16      // all-zero pad slots behind the 4 * Qp real ones (one per bank pair)

struct LowdegArgs {
    int n, Q, Qp, RT, LRT, C, W, R_real;
    int n4;                         // row pitch of best_states: 4 * Q
    uint32_t off_cnt, off_part, off_misc;      // (the pairs start at shared offset 0)
    float hK, knsh;
    int noise_on, maximize, use_target, n_sample_steps;
    long long step_begin, step_end, cadence, trace_stride;
    double target, w_total;
    const uint32_t *quad_of;        // [Qp] quad at a position; >= Q: none (ghost item)
    const uint4 *stream_w;          // N = 2: {ids 0|1, ids 2|3, f16 w 0|1, f16 w 2|3}
    const uint2 *stream_u;          // N = 3: {ids 0|1, ids 2|3}
    const int *warp_start;          // looped streams: first group row of each warp
    const float *hks_table;         // [steps + 1]  h ks(step) (x2 for N = 2), float64 on the host
    const uint64_t *seeds;          // [tiles * RT]
    const long long *sample_steps;  // global step indices after which a trace sample is taken
    float bnd[4];                   // N = 3: the float32 decision boundaries of the reference threshold rule
    double *io;                     // [R][n] phases in and out (float64, the reference's layout)
    double *best_obj, *energy, *best_trace;
    uint8_t *best_states;           // [tiles * RT][n4]
    long long *first_hit;
    unsigned long long *nonfinite;
};

__device__ __forceinline__ float xor_sign(float w, float c)       // w * sigma(c): flip w's sign where c's sign bit is set
{
    return __uint_as_float(__float_as_uint(w) ^ (__float_as_uint(c) & 0x80000000u));
}

// NMODE 2: OIM max-cut, integer couplings;  NMODE 3: OPM 3-colouring, unit couplings.
template <int NMODE, int QPT, bool UNIFORM>
__global__ void __launch_bounds__(QPT > 5 ? 512 : 1024, 1) k_lowdeg(const LowdegArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *cs = reinterpret_cast<float2 *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane & (a.RT - 1), c = lane >> a.LRT;
    const int tile = blockIdx.x, rg = tile * a.RT + r;
    const bool live = rg < a.R_real;
    const float2 *cs_lane = cs + r;                                  // + slot * RT
    const int WC = a.W * a.C;
    const int pos0 = warp * a.C + c;                                 // position of item 0; item t: + t * WC
    const uint32_t kstep = (uint32_t)a.Qp * a.RT;                    // pairs between component planes
    int *cnt = reinterpret_cast<int *>(smem_raw + a.off_cnt);
    double *part = reinterpret_cast<double *>(smem_raw + a.off_part);
    double *best_s = reinterpret_cast<double *>(smem_raw + a.off_misc);
    int *improved_s = reinterpret_cast<int *>(smem_raw + a.off_misc + a.RT * 8);

    // ---- prologue: the thread's items ------------------------------------------------------------
    uint32_t qid[QPT];
    float phi[QPT][4];
#pragma unroll
    for (int t = 0; t < QPT; ++t) {
        qid[t] = a.quad_of[pos0 + t * WC];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = 4u * qid[t] + k;
            phi[t][k] = (qid[t] < (uint32_t)a.Q && i < (uint32_t)a.n && live) ? (float)a.io[(size_t)rg * a.n + i] : 0.0f;
        }
    }
    const uint64_t seed = a.seeds[rg];
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    for (int i = tid; i < OSCB_LD_PADS * a.RT; i += blockDim.x) cs[(size_t)4 * kstep + i] = make_float2(0.0f, 0.0f);
    if (tid < a.RT) {
        best_s[tid] = a.best_obj[tile * a.RT + tid];
        improved_s[tid] = 0;
        cnt[tid] = 0;
    }

    // pass B: pairs of the phases in the registers -> the thread's own slots
    auto pass_b = [&]() {
#pragma unroll
        for (int t = 0; t < QPT; ++t) {
            float2 *own = cs + (size_t)(pos0 + t * WC) * a.RT + r;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float s, co;
                trig_turns_fast(phi[t][k], s, co);
                if (NMODE == 3) {
                    const float p = phi[t][k];
                    const uint32_t oh = (p >= a.bnd[0] && p < a.bnd[1]) ? 2u : ((p >= a.bnd[1] && p < a.bnd[2]) ? 4u : 1u);
                    co = __uint_as_float((__float_as_uint(co) & ~7u) | oh);
                }
                own[(size_t)k * kstep] = make_float2(co, s);
            }
        }
    };
    pass_b();
    __syncthreads();

    const uint4 *sw = a.stream_w + ((size_t)(UNIFORM ? warp * 4 : a.warp_start[warp]) * a.C + c);
    const uint2 *su = a.stream_u + ((size_t)(UNIFORM ? warp * 4 : a.warp_start[warp]) * a.C + c);
    const int W4C = a.W * 4 * a.C;

    // what the state now in shared memory still owes: a cadence score, or a trace sample (column >= 0)
    bool pending = true;
    int pending_col = 0;                 // the t = 0 sample (dynamics.py:385)
    long long pending_label = -1;
    int sample_cur = 0;
    while (sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] < a.step_begin) ++sample_cur;
    long long next_sample = sample_cur < a.n_sample_steps ? a.sample_steps[sample_cur] : -1;
    int cmod = a.cadence > 0 ? (int)(a.step_begin % a.cadence) : 1;

    // ---- pass A ------------------------------------------------------------------------------------
    // MODE 0: update only; 1: + read-out count; 2: + read-out count + energy; 3: count + energy, no update
    auto pass_a = [&](auto mode_tag, long long step, float hks) {
        constexpr int MODE = decltype(mode_tag)::value;
        float S = 0.0f;          // N = 2: sum_i sigma_i sum_j w_ij sigma_j (exact integer in float32)
        uint32_t same = 0;       // N = 3: equal-state neighbours
        double en = 0.0;         // (22 passes per run carry it)
        const uint4 *pw = sw;
        const uint2 *pu = su;
        uint4 curw = make_uint4(0, 0, 0, 0);
        uint2 curu = make_uint2(0, 0);
        if (!UNIFORM) {
            if (NMODE == 2) curw = *pw; else curu = *pu;
        }
#pragma unroll
        for (int t = 0; t < QPT; ++t) {
            float z[4] = {0.f, 0.f, 0.f, 0.f};
            if (MODE != 3 && a.noise_on)
                normals4_fast(philox4x32_10(make_uint4(qid[t], (uint32_t)step, (uint32_t)(step >> 32), 0x6F736362u), key),
                              z[0], z[1], z[2], z[3]);
            const float2 *own_p = cs_lane + (size_t)(pos0 + t * WC) * a.RT;
            float ynew[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 own = own_p[(size_t)k * kstep];
                const uint32_t ownmask = NMODE == 3 ? (__float_as_uint(own.x) & 7u) : 0u;
                float2 sum = make_float2(0.f, 0.f);
                float tsig = 0.f;
                uint32_t eq = 0;
                auto group = [&](uint32_t ix, uint32_t iy, uint32_t wx, uint32_t wy) {
                    const float2 v0 = cs_lane[ix & 0xffffu], v1 = cs_lane[ix >> 16];
                    const float2 v2 = cs_lane[iy & 0xffffu], v3 = cs_lane[UNIFORM ? (iy >> 16) : ((iy >> 16) & 0x7fffu)];
                    if (NMODE == 2) {
                        const float2 w01 = __half22float2(*reinterpret_cast<const __half2 *>(&wx));
                        const float2 w23 = __half22float2(*reinterpret_cast<const __half2 *>(&wy));
                        sum = __ffma2_rn(make_float2(w01.x, w01.x), v0, sum);
                        sum = __ffma2_rn(make_float2(w01.y, w01.y), v1, sum);
                        sum = __ffma2_rn(make_float2(w23.x, w23.x), v2, sum);
                        sum = __ffma2_rn(make_float2(w23.y, w23.y), v3, sum);
                        if (MODE >= 1)
                            tsig += (xor_sign(w01.x, v0.x) + xor_sign(w01.y, v1.x)) + (xor_sign(w23.x, v2.x) + xor_sign(w23.y, v3.x));
                    } else {
                        sum = __fadd2_rn(sum, __fadd2_rn(__fadd2_rn(v0, v1), __fadd2_rn(v2, v3)));
                        if (MODE >= 1)
                            eq += ((__float_as_uint(v0.x) & ownmask) + (__float_as_uint(v1.x) & ownmask)) +
                                  ((__float_as_uint(v2.x) & ownmask) + (__float_as_uint(v3.x) & ownmask));
                    }
                };
                if (UNIFORM) {
                    if (NMODE == 2) { const uint4 e = sw[(size_t)t * W4C + k * a.C]; group(e.x, e.y, e.z, e.w); }
                    else            { const uint2 e = su[(size_t)t * W4C + k * a.C]; group(e.x, e.y, 0, 0); }
                } else {
                    bool last;
                    do {
                        if (NMODE == 2) {
                            const uint4 e = curw;
                            pw += a.C;
                            curw = *pw;
                            last = (e.y >> 31) != 0;
                            group(e.x, e.y, e.z, e.w);
                        } else {
                            const uint2 e = curu;
                            pu += a.C;
                            curu = *pu;
                            last = (e.y >> 31) != 0;
                            group(e.x, e.y, 0, 0);
                        }
                    } while (!last);
                }
                if (MODE >= 1) {
                    if (NMODE == 2) S += xor_sign(tsig, own.x);
                    else same += eq >> (ownmask >> 1);
                }
                if (MODE >= 2) en += (double)own.x * (double)sum.x + (double)own.y * (double)sum.y;
                if (MODE != 3) {
                    const float acc = own.y * sum.x - own.x * sum.y;                 // dynamics.py:170
                    const float shil = NMODE == 2 ? own.y * own.x : own.y * (3.0f - 4.0f * own.y * own.y);
                    const float x = fmaf(a.hK, acc, fmaf(-hks, shil, fmaf(a.knsh, z[k], phi[t][k])));
                    const float w = x - floorf(x);                                   // dynamics.py:172
                    ynew[k] = (w >= 1.0f) ? 0.0f : w;
                }
            }
            if (MODE != 3) {
                const float chk = (ynew[0] + ynew[1]) + (ynew[2] + ynew[3]);     // NaN iff some x was not finite
                if (!(chk == chk) && live) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (!(ynew[k] == ynew[k])) flag_nonfinite(a.nonfinite, (uint64_t)step, (uint32_t)rg, 4u * qid[t] + k);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) phi[t][k] = ynew[k];
            }
        }
        if (MODE >= 1) {
            // read-out of the state that was in shared memory during this pass
            int v = NMODE == 2 ? __float2int_rn(S) : (int)same;
            for (int off = 16; off >= a.RT; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane < a.RT) atomicAdd(&cnt[lane], v);
            if (MODE >= 2) {
                double e = 0.5 * en;
                for (int off = 16; off >= a.RT; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
                if (lane < a.RT) part[warp * a.RT + lane] = e;
            }
            __syncthreads();
            if (tid < a.RT) {
                const int tot = cnt[tid];
                cnt[tid] = 0;
                const double obj = NMODE == 2 ? (a.w_total - (double)tot) * 0.25 : 0.5 * (double)tot;
                const double b = best_s[tid];
                const bool better = a.maximize ? (obj > b) : (obj < b);       // strict: dynamics.py:370-375
                improved_s[tid] = better ? 1 : 0;
                const int gi = tile * a.RT + tid;
                if (better) {
                    best_s[tid] = obj;
                    if (a.use_target && a.first_hit[gi] < 0 && (a.maximize ? (obj >= a.target) : (obj <= a.target)))
                        a.first_hit[gi] = pending_label;
                }
                if (MODE >= 2 && pending_col >= 0) {
                    double en_tot = 0.0;
                    for (int w = 0; w < a.W; ++w) en_tot += part[w * a.RT + tid];      // fixed order: deterministic trace
                    a.energy[(size_t)gi * a.trace_stride + pending_col] = en_tot;
                    a.best_trace[(size_t)gi * a.trace_stride + pending_col] = best_s[tid];
                }
            }
            __syncthreads();
            if (improved_s[r] && live) {
                // the pairs in shared memory still are the scored state: its lattice states -> best_states
#pragma unroll
                for (int t = 0; t < QPT; ++t) {
                    if (qid[t] < (uint32_t)a.Q) {
                        const float2 *own_p = cs_lane + (size_t)(pos0 + t * WC) * a.RT;
                        uint32_t packed = 0;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t bits = __float_as_uint(own_p[(size_t)k * kstep].x);
                            const uint32_t st = NMODE == 2 ? (bits >> 31) : ((bits & 7u) >> 1);
                            packed |= st << (8 * k);
                        }
                        *reinterpret_cast<uint32_t *>(a.best_states + (size_t)rg * a.n4 + 4u * qid[t]) = packed;
                    }
                }
            }
        }
    };
    using M0 = std::integral_constant<int, 0>;
    using M1 = std::integral_constant<int, 1>;
    using M2 = std::integral_constant<int, 2>;
    using M3 = std::integral_constant<int, 3>;

    // ---- time loop ---------------------------------------------------------------------------------
#pragma unroll 1
    for (long long step = a.step_begin; step < a.step_end; ++step) {
        const float hks = __ldg(a.hks_table + (step - a.step_begin));
        if (!pending) {
            pass_a(M0{}, step, hks);
            __syncthreads();
        } else if (pending_col < 0) {
            pass_a(M1{}, step, hks);         // (ends behind a barrier of its own; publishing reads own slots only)
        } else {
            pass_a(M2{}, step, hks);
        }
        pending = false;
        pass_b();
        __syncthreads();
        const bool is_sample = step == next_sample;
        const bool cadence_hit = a.cadence > 0 && cmod == 0;
        cmod = (cmod + 1 == (int)a.cadence) ? 0 : cmod + 1;
        if (is_sample) {
            pending = true;
            pending_col = 1 + sample_cur;
            pending_label = step;
            ++sample_cur;
            next_sample = sample_cur < a.n_sample_steps ? a.sample_steps[sample_cur] : -1;
        } else if (cadence_hit) {
            pending = true;
            pending_col = -1;
            pending_label = step;
        }
    }
    if (pending) pass_a(M3{}, a.step_end, 0.0f);

    if (tid < a.RT) a.best_obj[tile * a.RT + tid] = best_s[tid];
    if (live) {
#pragma unroll
        for (int t = 0; t < QPT; ++t)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t i = 4u * qid[t] + k;
                if (qid[t] < (uint32_t)a.Q && i < (uint32_t)a.n) a.io[(size_t)rg * a.n + i] = (double)phi[t][k];
            }
    }
}

} // namespace oscb
