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
//     that uses it, coalesced: 4 x u32 BYTE OFFSETS of the neighbours' slots (no unpacking, no address
//     arithmetic: with one replica per CTA the offset is the LDS address) and, for N = 2, 4 x f32 couplings
//     (unit weights are the same stream with 1.0; padding reads an all-zero slot with coupling 0).  UNIFORM
//     graphs (every row <= 4 neighbours) have exactly one group per row at an address known at compile time up
//     to a stride -- straight-line code; otherwise a warp walks its groups with a running pointer and a "last
//     group of the row" flag in bit 31 of the group's fourth offset;
//   * read-out rides on the gather of the NEXT step (as in k_resident_fast): for N = 2 the sign bit of a stored
//     cosine is the oscillator's lattice state, and cut = (W - sum_i sigma_i sum_j w_ij sigma_j) / 4 needs one
//     LOP3 + one FADD per neighbour; for N = 3 the low three mantissa bits of the stored cosine hold the
//     state one-hot (a <= 7 ulp perturbation of a value whose own MUFU error is larger), so the count of
//     equal-state neighbours is one AND + one add per neighbour.  Trace samples ride the same way, the
//     energy being sum_i (c_i, s_i) . sum_j w_ij (c_j, s_j) / 2 of the gather sums that are there anyway.
//
// Arithmetic of a step (float32, FMA-contracted) is k_resident_fast's; parity is by tolerance and distribution.
#pragma once
#include "oscb_fastmath.cuh"

namespace oscb {

#define OSCB_LD_TAB 192       // most CTAs of one launch of a mixed-tile schedule
#define OSCB_LD_PADS 16      // all-zero pad slots behind the 4 * Qp real ones (one per bank pair)

struct LowdegArgs {
    int n, Q, Qp, RT, LRT, C, W, R_real;
    int n4;                         // row pitch of best_states: 4 * Q
    uint32_t off_cnt, off_part, off_misc;      // (the pairs start at shared offset 0)
    uint32_t off_ids, n_ids;                   // k_lowdeg_pair with its slot stream staged in shared memory: offset, entries (uint2)
    float hK, knsh;
    int noise_on, maximize, use_target, n_sample_steps;
    int step_begin, step_end, cadence;
    long long trace_stride;
    double target, w_total;
    const uint32_t *quad_of;        // [Qp] quad at a position; >= Q: none (ghost item)
    const uint4 *soff;              // byte offsets of a group's four neighbour slots (replica 0 of the tile)
    const uint2 *sidx;              // k_lowdeg_pair: the same groups as 4 x u16 SLOT numbers
    const uint32_t *row_groups;     // k_lowdeg_pair: [W][QPT] group counts of an item's four rows in visiting order, a byte each
    // one window of a mixed-tile schedule (use_tab = 0: CTA b is tile b and runs [step_begin, step_end)): CTA b integrates tile
    // tab_tile[b] (of RT replicas) over [win_begin, win_begin + window_steps) (hks_table stays indexed from step_begin).  All
    // CTAs of a launch share the window -- tiles with another history get a launch of their own -- so the step counter and
    // all that hangs on it (Philox counter, schedule look-up, cadence) stay on the uniform datapath as in the unbroken launch
    // (with a per-CTA first step k_lowdeg needed 63 registers instead of 56 and lost 6 %).  The table travels in the
    // kernel parameters.
    int use_tab, win_begin, window_steps;
    int tab_tile[OSCB_LD_TAB];
    const float4 *swt;              // N = 2: their couplings
    const int *warp_start;          // looped streams: first group row of each warp
    const float *hks_table;         // [steps + 1]  h ks(step) (x2 for N = 2), float64 on the host
    const uint64_t *seeds;          // [tiles * RT]
    const int *sample_steps;        // global step indices after which a trace sample is taken
    float bnd[4];                   // N = 3: the float32 decision boundaries of the reference threshold rule
    double *io;                     // [R][n] phases in and out (float64, the reference's layout)
    double *best_obj, *energy, *best_trace;
    uint8_t *best_states;           // [tiles * RT][n4]
    long long *first_hit;
    unsigned long long *nonfinite;
};

// threads per CTA by items per thread: the phases of QPT quads stay in registers, so more items need more registers
// per thread (64 / 80 / 128)
__host__ __device__ constexpr int lowdeg_max_threads(int qpt) { return qpt <= 4 ? 1024 : (qpt <= 7 ? 768 : 512); }
// k_lowdeg_pair holds two replicas per lane: from two items per thread on it wants the 128 registers of a 512-thread CTA
__host__ __device__ constexpr int lowdeg_pair_max_threads(int qpt) { return qpt <= 1 ? 1024 : 512; }

// x - floor(x) on the FMA/ALU pipes for |x| < 2^22 (the conversion unit is as busy as the MUFU unit here): the
// magic-number add rounds x to the nearest integer, a compare steps it down to the floor.  Anything larger (or
// non-finite) takes floorf.  Same value as x - floorf(x) for every x (both subtractions are exact or round once).
__device__ __forceinline__ float frac_alu(float x)          // |x| < 2^22
{
    const float r = (x + 12582912.0f) - 12582912.0f;        // rint(x)
    const float f = r - (r > x ? 1.0f : 0.0f);              // floor(x)
    return x - f;
}

__device__ __forceinline__ float xor_sign(float w, float c)       // w * sigma(c): flip w's sign where c's sign bit is set
{
    return __uint_as_float(__float_as_uint(w) ^ (__float_as_uint(c) & 0x80000000u));
}

// NMODE 2: OIM max-cut, integer couplings;  NMODE 3: OPM 3-colouring, unit couplings.
// RT1: one replica per CTA (a slot offset IS the shared-memory address of the pair).
// WIN: one window of a mixed-tile schedule (the per-CTA table of LowdegArgs); a separate instantiation, so that the unbroken
// launch keeps its code (with the table read behind a run-time flag the flat200 kernel lost 6 %).
template <int NMODE, int QPT, bool UNIFORM, bool RT1, bool WIN = false>
__global__ void __launch_bounds__(lowdeg_max_threads(QPT), 1) k_lowdeg(const LowdegArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = RT1 ? 0 : (lane & (a.RT - 1)), c = RT1 ? lane : (lane >> a.LRT);
    // One window of a mixed-tile schedule: the tile and its first step come from the per-CTA table in the parameters (see
    // LowdegArgs), re-read where needed instead of being held: this kernel has no register to spare (64 at 1024 threads).
    auto tile_now = [&]() -> int { return WIN ? a.tab_tile[blockIdx.x] : (int)blockIdx.x; };
    auto end_step = [&]() -> int { return WIN ? a.win_begin + a.window_steps : a.step_end; };
    const int sb = WIN ? a.win_begin : a.step_begin;
    const bool live = tile_now() * a.RT + r < a.R_real;
    const unsigned char *cs_lane = smem_raw + r * 8;                 // + slot byte offset
    const int WC = a.W * a.C;
    const int pos0 = warp * a.C + c;                                 // position of item 0; item t: + t * WC
    const uint32_t kbytes = (uint32_t)a.Qp * a.RT * 8;               // bytes between component planes
    const uint32_t tbytes = (uint32_t)WC * a.RT * 8;                 // bytes between the items of a thread
    const uint32_t own0 = (uint32_t)(pos0 * a.RT + r) * 8;           // own slot of (item 0, component 0)
    int *cnt = reinterpret_cast<int *>(smem_raw + a.off_cnt);
    double *part = reinterpret_cast<double *>(smem_raw + a.off_part);
    double *best_s = reinterpret_cast<double *>(smem_raw + a.off_misc);
    int *improved_s = reinterpret_cast<int *>(smem_raw + a.off_misc + a.RT * 8);
    auto pair_at = [&](uint32_t off) -> float2 {
        return *reinterpret_cast<const float2 *>((RT1 ? smem_raw : cs_lane) + off);
    };

    // ---- prologue: the thread's items ------------------------------------------------------------
    // the quad of item t: its position itself on uniform graphs (natural order), else looked up (L1/L2) when needed
    auto quad = [&](int t) -> uint32_t { return UNIFORM ? (uint32_t)(pos0 + t * WC) : __ldg(a.quad_of + pos0 + t * WC); };
    float phi[QPT][4];
#pragma unroll
    for (int t = 0; t < QPT; ++t) {
        const uint32_t q = quad(t);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = 4u * q + k;
            phi[t][k] = (q < (uint32_t)a.Q && i < (uint32_t)a.n && live) ? (float)a.io[(size_t)(tile_now() * a.RT + r) * a.n + i] : 0.0f;
        }
    }
    const uint64_t seed = a.seeds[tile_now() * a.RT + r];
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    for (int i = tid; i < OSCB_LD_PADS * a.RT; i += blockDim.x)
        reinterpret_cast<float2 *>(smem_raw + (size_t)4 * kbytes)[i] = make_float2(0.0f, 0.0f);
    if (tid < a.RT) {
        best_s[tid] = a.best_obj[tile_now() * a.RT + tid];
        improved_s[tid] = 0;
        cnt[tid] = 0;
    }

    // pass B: pairs of the phases in the registers -> the thread's own slots
    // `with_state`: the next pass A reads lattice states out of these pairs.  N = 2 always carries the state (it is the
    // cosine's sign bit, three instructions); the N = 3 one-hot bits cost six and are written only when they will be read.
    const float b0 = a.bnd[0], b1 = a.bnd[1], b2 = a.bnd[2];
    auto pass_b = [&](bool with_state) {
#pragma unroll
        for (int t = 0; t < QPT; ++t) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float s, co;
                trig_turns_direct(phi[t][k], s, co);
                if (NMODE == 3 && with_state) {
                    const float p = phi[t][k];
                    uint32_t oh = p >= b0 ? 2u : 1u;
                    oh = p >= b1 ? 4u : oh;
                    oh = p >= b2 ? 1u : oh;
                    co = __uint_as_float((__float_as_uint(co) & ~7u) | oh);
                }
                *reinterpret_cast<float2 *>(smem_raw + own0 + t * tbytes + k * kbytes) = make_float2(co, s);
            }
        }
    };
    pass_b(true);
    __syncthreads();

    const size_t first_row = UNIFORM ? (size_t)warp * 4 : (size_t)a.warp_start[warp];
    const uint4 *so = a.soff + first_row * a.C + c;
    const float4 *sw = a.swt + first_row * a.C + c;
    const int W4C = a.W * 4 * a.C;

    // what the state now in shared memory still owes: a cadence score, or a trace sample (column >= 0)
    bool pending = WIN ? sb == a.step_begin : true;
    int pending_col = 0;                 // the t = 0 sample (dynamics.py:385)
    int pending_label = -1;
    int sample_cur = 0;
    while (sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] < sb) ++sample_cur;
    int next_sample = sample_cur < a.n_sample_steps ? a.sample_steps[sample_cur] : -1;
    int cmod = a.cadence > 0 ? sb % a.cadence : 1;

    // ---- pass A ------------------------------------------------------------------------------------
    // MODE 0: update only; 1: + read-out count; 2: + read-out count + energy; 3: count + energy, no update
    auto pass_a = [&](auto mode_tag, int step, float hks) {
        constexpr int MODE = decltype(mode_tag)::value;
        float S = 0.0f;          // N = 2: sum_i sigma_i sum_j w_ij sigma_j (exact integer in float32)
        uint32_t same = 0;       // N = 3: equal-state neighbours
        double en = 0.0;         // (22 passes per run carry it)
        bool bad = false;
        const uint4 *po = so;
        const float4 *pw = sw;
        const int stride = a.C;
#pragma unroll
        for (int t = 0; t < QPT; ++t) {
            float z[4] = {0.f, 0.f, 0.f, 0.f};
            if (MODE != 3 && a.noise_on)
                normals4_fast(philox4x32_10(make_uint4(quad(t), (uint32_t)step, 0u, 0x6F736362u), key), z[0], z[1], z[2], z[3]);
            float ynew[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 own = *reinterpret_cast<const float2 *>(smem_raw + own0 + t * tbytes + k * kbytes);
                const uint32_t ownmask = NMODE == 3 ? (__float_as_uint(own.x) & 7u) : 0u;
                float2 sum = make_float2(0.f, 0.f);
                float tsig = 0.f;
                uint32_t eq = 0;
                auto group = [&](const uint4 o, const float4 w) {
                    const float2 v0 = pair_at(o.x), v1 = pair_at(o.y), v2 = pair_at(o.z);
                    const float2 v3 = pair_at(UNIFORM ? o.w : (o.w & 0x7fffffffu));
                    if (NMODE == 2) {
                        sum = __ffma2_rn(make_float2(w.x, w.x), v0, sum);
                        sum = __ffma2_rn(make_float2(w.y, w.y), v1, sum);
                        sum = __ffma2_rn(make_float2(w.z, w.z), v2, sum);
                        sum = __ffma2_rn(make_float2(w.w, w.w), v3, sum);
                        if (MODE >= 1)
                            tsig += (xor_sign(w.x, v0.x) + xor_sign(w.y, v1.x)) + (xor_sign(w.z, v2.x) + xor_sign(w.w, v3.x));
                    } else {
                        sum = __fadd2_rn(sum, __fadd2_rn(__fadd2_rn(v0, v1), __fadd2_rn(v2, v3)));
                        if (MODE >= 1)
                            eq += ((__float_as_uint(v0.x) & ownmask) + (__float_as_uint(v1.x) & ownmask)) +
                                  ((__float_as_uint(v2.x) & ownmask) + (__float_as_uint(v3.x) & ownmask));
                    }
                };
                if (UNIFORM) {
                    const int e = t * W4C + k * a.C;
                    group(__ldcg(so + e), NMODE == 2 ? __ldcg(sw + e) : make_float4(0.f, 0.f, 0.f, 0.f));
                } else {
                    // (no software prefetch: the stream sits in L1 / L2 and the other warps cover the load; carrying the next
                    // group in registers cost four moves per group)
                    bool last;
                    do {
                        const uint4 o = __ldg(po);
                        const float4 w = NMODE == 2 ? __ldg(pw) : make_float4(0.f, 0.f, 0.f, 0.f);
                        po += stride;
                        if (NMODE == 2) pw += stride;
                        // (the flag is the same in all lanes: the vote tells the compiler so -- a uniform branch, no
                        // reconvergence bookkeeping around every row)
                        last = __any_sync(0xffffffffu, (int)o.w < 0);
                        group(o, w);
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
                    ynew[k] = x;
                }
            }
            if (MODE != 3) {
                // wrap (dynamics.py:172).  N = 2 (the G81 shape: the MUFU / conversion unit is the busy one): on the ALU, one
                // range check per quad, a huge or non-finite x takes floorf; N = 3: floorf (fewer instructions, the unit has room)
                const float big = fmaxf(fmaxf(fabsf(ynew[0]), fabsf(ynew[1])), fmaxf(fabsf(ynew[2]), fabsf(ynew[3])));
                const float any = (ynew[0] + ynew[1]) + (ynew[2] + ynew[3]);     // NaN iff some x is NaN (fmaxf drops NaNs)
                if (NMODE == 2 && big < 4194304.0f && any == any) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float w = frac_alu(ynew[k]);
                        ynew[k] = (w >= 1.0f) ? 0.0f : w;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float w = ynew[k] - floorf(ynew[k]);
                        ynew[k] = (w >= 1.0f) ? 0.0f : w;
                    }
                }
                const float chk = (ynew[0] + ynew[1]) + (ynew[2] + ynew[3]);     // NaN iff some x was not finite
                bad = bad || !(chk == chk);
#pragma unroll
                for (int k = 0; k < 4; ++k) phi[t][k] = ynew[k];
            }
        }
        if (MODE != 3 && bad && live) {
            // a non-finite x leaves a NaN phase behind: name the first ones (dynamics.py:276-283)
#pragma unroll
            for (int t = 0; t < QPT; ++t)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (!(phi[t][k] == phi[t][k]) && quad(t) < (uint32_t)a.Q)
                        flag_nonfinite(a.nonfinite, (uint64_t)step, (uint32_t)(tile_now() * a.RT + r), 4u * quad(t) + k);
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
                const int gi = tile_now() * a.RT + tid;
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
                    const uint32_t q = quad(t);
                    if (q < (uint32_t)a.Q) {
                        uint32_t packed = 0;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t bits = __float_as_uint(reinterpret_cast<const float2 *>(smem_raw + own0 + t * tbytes + k * kbytes)->x);
                            const uint32_t st = NMODE == 2 ? (bits >> 31) : ((bits & 7u) >> 1);
                            packed |= st << (8 * k);
                        }
                        *reinterpret_cast<uint32_t *>(a.best_states + (size_t)(tile_now() * a.RT + r) * a.n4 + 4u * q) = packed;
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
    for (int step = sb; step < end_step(); ++step) {
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
        const bool is_sample = step == next_sample;
        const bool cadence_hit = a.cadence > 0 && cmod == 0;
        pass_b(is_sample || cadence_hit);
        __syncthreads();
        cmod = (cmod + 1 == a.cadence) ? 0 : cmod + 1;
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
    if (pending) pass_a(M3{}, end_step(), 0.0f);

    if (tid < a.RT) a.best_obj[tile_now() * a.RT + tid] = best_s[tid];
    if (live) {
#pragma unroll
        for (int t = 0; t < QPT; ++t) {
            const uint32_t q = quad(t);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t i = 4u * q + k;
                if (q < (uint32_t)a.Q && i < (uint32_t)a.n) a.io[(size_t)(tile_now() * a.RT + r) * a.n + i] = (double)phi[t][k];
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------------------------
// k_lowdeg_pair -- the same register-resident design for N = 2 max-cut at ANY degree, two replicas per lane.
//
// k_resident_fast spends more on a row's bookkeeping (row table, group counts, phases through L2, staged pairs, a
// pass-B copy: ~100 lane-instructions per replica-oscillator on the G22 shape) than on its 20 gathers (~78).  Here the
// per-oscillator part is k_lowdeg's (phases in registers, trig after the barrier, ~30), and the gather keeps what makes
// k_resident_fast's cheap: a lane owns TWO adjacent replicas, so one LDS.128 fetches both (cos, sin) pairs of a
// neighbour and the stream words, the address add and the loop control are shared by two updates.  Looped stream
// only (rows of any degree); UNITW: unit couplings -- plain packed adds, and the coupling stream is read only on the
// steps that read the cut out (it carries the zeros that keep padding out of the count).
// IDS: the slot stream is staged in shared memory behind the pairs (when both fit: G22 shape, 8 replicas: 129 + 95 KB), so
// a group's slot numbers come back in an LDS latency instead of an L1 / L2 one.
template <int QPT, bool UNITW, bool IDS>
__global__ void __launch_bounds__(lowdeg_pair_max_threads(QPT), 1) k_lowdeg_pair(const LowdegArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int LPS = a.RT >> 1;                                       // lanes per slot
    const int q = lane & (LPS - 1), c = lane >> (a.LRT - 1);
    const int r0 = 2 * q;
    const int tile = a.use_tab ? a.tab_tile[blockIdx.x] : (int)blockIdx.x, rg0 = tile * a.RT + r0;
    const int sb = a.use_tab ? a.win_begin : a.step_begin, se = a.use_tab ? sb + a.window_steps : a.step_end;
    const bool live[2] = {rg0 < a.R_real, rg0 + 1 < a.R_real};
    const unsigned char *cs_lane = smem_raw + r0 * 8;                // + slot byte offset: the pairs of replicas r0, r0 + 1
    const int WC = a.W * a.C;
    const int pos0 = warp * a.C + c;
    const uint32_t kbytes = (uint32_t)a.Qp * a.RT * 8;
    const uint32_t tbytes = (uint32_t)WC * a.RT * 8;
    const uint32_t own0 = (uint32_t)(pos0 * a.RT + r0) * 8;
    int *cnt = reinterpret_cast<int *>(smem_raw + a.off_cnt);
    double *part = reinterpret_cast<double *>(smem_raw + a.off_part);
    double *best_s = reinterpret_cast<double *>(smem_raw + a.off_misc);
    int *improved_s = reinterpret_cast<int *>(smem_raw + a.off_misc + a.RT * 8);
    // (c0, s0, c1, s1) of the two replicas of this lane at a slot
    const uint32_t slot_bytes = (uint32_t)a.RT * 8u;
    auto pairs_at = [&](uint32_t slot) -> float4 { return *reinterpret_cast<const float4 *>(cs_lane + slot * slot_bytes); };
    // quad table word: quad number (24 bits, all ones = ghost) | the components of its rows in visiting order (4 x 2 bits)
    auto quad = [&](int t) -> uint32_t { return __ldg(a.quad_of + pos0 + t * WC); };
    auto comp_of = [](uint32_t qw, int k) -> uint32_t { return (qw >> (24 + 2 * k)) & 3u; };

    float phi[QPT][4][2];
#pragma unroll
    for (int t = 0; t < QPT; ++t) {
        const uint32_t qw = quad(t), qd = qw & 0xFFFFFFu;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = 4u * qd + comp_of(qw, k);
#pragma unroll
            for (int e = 0; e < 2; ++e)
                phi[t][k][e] = (qd < (uint32_t)a.Q && i < (uint32_t)a.n && live[e]) ? (float)a.io[(size_t)(rg0 + e) * a.n + i] : 0.0f;
        }
    }
    uint2 key[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const uint64_t seed = a.seeds[rg0 + e];
        key[e] = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    }
    for (int i = tid; i < OSCB_LD_PADS * a.RT; i += blockDim.x)
        reinterpret_cast<float2 *>(smem_raw + (size_t)4 * kbytes)[i] = make_float2(0.0f, 0.0f);
    if (tid < a.RT) {
        best_s[tid] = a.best_obj[tile * a.RT + tid];
        improved_s[tid] = 0;
        cnt[tid] = 0;
    }
    auto pass_b = [&]() {
#pragma unroll
        for (int t = 0; t < QPT; ++t)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float s0, c0, s1, c1;
                trig_turns_direct(phi[t][k][0], s0, c0);
                trig_turns_direct(phi[t][k][1], s1, c1);
                *reinterpret_cast<float4 *>(smem_raw + own0 + t * tbytes + k * kbytes) = make_float4(c0, s0, c1, s1);
            }
    };
    pass_b();
    if (IDS) {
        uint2 *dst = reinterpret_cast<uint2 *>(smem_raw + a.off_ids);
        for (uint32_t i = tid; i < a.n_ids; i += blockDim.x) dst[i] = __ldg(a.sidx + i);
    }
    __syncthreads();

    const size_t first_row = (size_t)a.warp_start[warp];
    // the stream as u16 slot numbers: 8 B per group, ~100 KB per step on the G22 shape -- it stays in the L1 the 132 KB
    // shared-memory configuration leaves (the u32-offset form, 200 KB, thrashed it: every group waited on L2)
    const uint2 *so = (IDS ? reinterpret_cast<const uint2 *>(smem_raw + a.off_ids) : a.sidx) + first_row * a.C + c;
    const float4 *sw = a.swt + first_row * a.C + c;

    bool pending = sb == a.step_begin;        // the read-out of the state the run starts from (a later window of a schedule: none)
    int pending_col = 0, pending_label = -1, sample_cur = 0;
    while (sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] < sb) ++sample_cur;
    int next_sample = sample_cur < a.n_sample_steps ? a.sample_steps[sample_cur] : -1;
    int cmod = a.cadence > 0 ? sb % a.cadence : 1;

    auto pass_a = [&](auto mode_tag, int step, float hks) {
        constexpr int MODE = decltype(mode_tag)::value;
        constexpr bool USE_W = !UNITW || MODE >= 1;
        float S[2] = {0.f, 0.f};
        double en[2] = {0.0, 0.0};
        bool bad = false;
        const uint2 *po = so;
        const float4 *pw = sw;
        const int stride = a.C;
        uint2 nxt = IDS ? *po : __ldg(po);   // the slot numbers run one group ahead of their use (the last group of a warp's
                                             // stream prefetches the pad row behind it)
#pragma unroll
        for (int t = 0; t < QPT; ++t) {
            float z[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
            if (MODE != 3 && a.noise_on) {
                const uint32_t qw = quad(t), qd = qw & 0xFFFFFFu;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    float n0, n1, n2, n3;
                    normals4_fast(philox4x32_10(make_uint4(qd, (uint32_t)step, 0u, 0x6F736362u), key[e]), n0, n1, n2, n3);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {                       // the k-th row visited is component comp_of(qw, k)
                        const uint32_t cm = comp_of(qw, k);
                        const float lo = (cm & 1u) ? n1 : n0, hi = (cm & 1u) ? n3 : n2;
                        z[e][k] = (cm & 2u) ? hi : lo;
                    }
                }
            }
            float ynew[4][2];
            const uint32_t gcount = __ldg(a.row_groups + warp * QPT + t);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float4 own = *reinterpret_cast<const float4 *>(smem_raw + own0 + t * tbytes + k * kbytes);
                float2 sum0 = make_float2(0.f, 0.f), sum1 = make_float2(0.f, 0.f);
                float ts0 = 0.f, ts1 = 0.f;
                // The adds of a group run one group behind its loads: while the four LDS.128 of group g are in flight the
                // packed adds of group g - 1 issue (a warp issues in order, so without this every group paid the full
                // shared-memory latency before its first add).  The first group is peeled: nothing to add behind it.
                float4 p0, p1, p2, p3, pwt = make_float4(1.f, 1.f, 1.f, 1.f);
                auto accumulate = [&](const float4 &v0, const float4 &v1, const float4 &v2, const float4 &v3, const float4 &w) {
                    if (USE_W) {
                        sum0 = __ffma2_rn(make_float2(w.x, w.x), make_float2(v0.x, v0.y), sum0);
                        sum1 = __ffma2_rn(make_float2(w.x, w.x), make_float2(v0.z, v0.w), sum1);
                        sum0 = __ffma2_rn(make_float2(w.y, w.y), make_float2(v1.x, v1.y), sum0);
                        sum1 = __ffma2_rn(make_float2(w.y, w.y), make_float2(v1.z, v1.w), sum1);
                        sum0 = __ffma2_rn(make_float2(w.z, w.z), make_float2(v2.x, v2.y), sum0);
                        sum1 = __ffma2_rn(make_float2(w.z, w.z), make_float2(v2.z, v2.w), sum1);
                        sum0 = __ffma2_rn(make_float2(w.w, w.w), make_float2(v3.x, v3.y), sum0);
                        sum1 = __ffma2_rn(make_float2(w.w, w.w), make_float2(v3.z, v3.w), sum1);
                    } else {
                        sum0 = __fadd2_rn(sum0, __fadd2_rn(__fadd2_rn(make_float2(v0.x, v0.y), make_float2(v1.x, v1.y)),
                                                           __fadd2_rn(make_float2(v2.x, v2.y), make_float2(v3.x, v3.y))));
                        sum1 = __fadd2_rn(sum1, __fadd2_rn(__fadd2_rn(make_float2(v0.z, v0.w), make_float2(v1.z, v1.w)),
                                                           __fadd2_rn(make_float2(v2.z, v2.w), make_float2(v3.z, v3.w))));
                    }
                    if (MODE >= 1) {
                        ts0 += (xor_sign(w.x, v0.x) + xor_sign(w.y, v1.x)) + (xor_sign(w.z, v2.x) + xor_sign(w.w, v3.x));
                        ts1 += (xor_sign(w.x, v0.z) + xor_sign(w.y, v1.z)) + (xor_sign(w.z, v2.z) + xor_sign(w.w, v3.z));
                    }
                };
                // one group's loads: its slot numbers were fetched a group ahead, the next group's are fetched now (the last
                // group of a warp's stream prefetches the pad row behind it)
                auto fetch = [&](float4 &v0, float4 &v1, float4 &v2, float4 &v3, float4 &w) {
                    const uint2 o = nxt;
                    po += stride;
                    nxt = IDS ? *po : __ldg(po);
                    if (USE_W) { w = __ldg(pw); }
                    pw += stride;
                    v0 = pairs_at(o.x & 0xffffu); v1 = pairs_at(o.x >> 16);
                    v2 = pairs_at(o.y & 0xffffu); v3 = pairs_at(o.y >> 16);
                };
                // the row's group count is warp-uniform and known up front: a counted loop, no vote per group
                const int G = (int)((gcount >> (8 * k)) & 0xffu);
                fetch(p0, p1, p2, p3, pwt);
#pragma unroll 2
                for (int g = 1; g < G; ++g) {
                    float4 v0, v1, v2, v3, w = make_float4(1.f, 1.f, 1.f, 1.f);
                    fetch(v0, v1, v2, v3, w);
                    accumulate(p0, p1, p2, p3, pwt);
                    p0 = v0; p1 = v1; p2 = v2; p3 = v3; pwt = w;
                }
                accumulate(p0, p1, p2, p3, pwt);
                if (MODE >= 1) { S[0] += xor_sign(ts0, own.x); S[1] += xor_sign(ts1, own.z); }
                if (MODE >= 2) {
                    en[0] += (double)own.x * (double)sum0.x + (double)own.y * (double)sum0.y;
                    en[1] += (double)own.z * (double)sum1.x + (double)own.w * (double)sum1.y;
                }
                if (MODE != 3) {
                    const float acc0 = own.y * sum0.x - own.x * sum0.y, acc1 = own.w * sum1.x - own.z * sum1.y;   // dynamics.py:170
                    ynew[k][0] = fmaf(a.hK, acc0, fmaf(-hks, own.y * own.x, fmaf(a.knsh, z[0][k], phi[t][k][0])));
                    ynew[k][1] = fmaf(a.hK, acc1, fmaf(-hks, own.w * own.z, fmaf(a.knsh, z[1][k], phi[t][k][1])));
                }
            }
            if (MODE != 3) {
                float chk = 0.f;
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const float w = ynew[k][e] - floorf(ynew[k][e]);                  // dynamics.py:172
                        const float y = (w >= 1.0f) ? 0.0f : w;
                        phi[t][k][e] = y;
                        chk += y;
                    }
                bad = bad || !(chk == chk);
            }
        }
        if (MODE != 3 && bad) {
#pragma unroll
            for (int t = 0; t < QPT; ++t)
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (!(phi[t][k][e] == phi[t][k][e]) && live[e] && (quad(t) & 0xFFFFFFu) < (uint32_t)a.Q)
                            flag_nonfinite(a.nonfinite, (uint64_t)step, (uint32_t)(rg0 + e), 4u * (quad(t) & 0xFFFFFFu) + comp_of(quad(t), k));
        }
        if (MODE >= 1) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                int v = __float2int_rn(S[e]);
                for (int off = 16; off >= LPS; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane < LPS) atomicAdd(&cnt[2 * lane + e], v);
                if (MODE >= 2) {
                    double x = 0.5 * en[e];
                    for (int off = 16; off >= LPS; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
                    if (lane < LPS) part[warp * a.RT + 2 * lane + e] = x;
                }
            }
            __syncthreads();
            if (tid < a.RT) {
                const int tot = cnt[tid];
                cnt[tid] = 0;
                const double obj = (a.w_total - (double)tot) * 0.25;
                const double b = best_s[tid];
                const bool better = obj > b;                                  // strict: dynamics.py:370-375
                improved_s[tid] = better ? 1 : 0;
                const int gi = tile * a.RT + tid;
                if (better) {
                    best_s[tid] = obj;
                    if (a.use_target && a.first_hit[gi] < 0 && obj >= a.target) a.first_hit[gi] = pending_label;
                }
                if (MODE >= 2 && pending_col >= 0) {
                    double en_tot = 0.0;
                    for (int w = 0; w < a.W; ++w) en_tot += part[w * a.RT + tid];
                    a.energy[(size_t)gi * a.trace_stride + pending_col] = en_tot;
                    a.best_trace[(size_t)gi * a.trace_stride + pending_col] = best_s[tid];
                }
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (improved_s[r0 + e] && live[e]) {
#pragma unroll
                    for (int t = 0; t < QPT; ++t) {
                        const uint32_t qw = quad(t), qd = qw & 0xFFFFFFu;
                        if (qd < (uint32_t)a.Q) {
                            uint32_t packed = 0;
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const float4 own = *reinterpret_cast<const float4 *>(smem_raw + own0 + t * tbytes + k * kbytes);
                                packed |= (__float_as_uint(e ? own.z : own.x) >> 31) << (8 * comp_of(qw, k));
                            }
                            *reinterpret_cast<uint32_t *>(a.best_states + (size_t)(rg0 + e) * a.n4 + 4u * qd) = packed;
                        }
                    }
                }
            }
        }
    };
    using M0 = std::integral_constant<int, 0>;
    using M1 = std::integral_constant<int, 1>;
    using M2 = std::integral_constant<int, 2>;
    using M3 = std::integral_constant<int, 3>;
#pragma unroll 1
    for (int step = sb; step < se; ++step) {
        const float hks = __ldg(a.hks_table + (step - a.step_begin));
        if (!pending) {
            pass_a(M0{}, step, hks);
            __syncthreads();
        } else if (pending_col < 0) {
            pass_a(M1{}, step, hks);
        } else {
            pass_a(M2{}, step, hks);
        }
        pending = false;
        pass_b();
        __syncthreads();
        const bool is_sample = step == next_sample;
        const bool cadence_hit = a.cadence > 0 && cmod == 0;
        cmod = (cmod + 1 == a.cadence) ? 0 : cmod + 1;
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
    if (pending) pass_a(M3{}, se, 0.0f);

    if (tid < a.RT) a.best_obj[tile * a.RT + tid] = best_s[tid];
#pragma unroll
    for (int t = 0; t < QPT; ++t) {
        const uint32_t qw = quad(t), qd = qw & 0xFFFFFFu;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = 4u * qd + comp_of(qw, k);
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (live[e] && qd < (uint32_t)a.Q && i < (uint32_t)a.n) a.io[(size_t)(rg0 + e) * a.n + i] = (double)phi[t][k][e];
        }
    }
}


} // namespace oscb
