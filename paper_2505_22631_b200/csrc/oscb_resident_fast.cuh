// oscb_resident_fast.cuh -- the production (float32) variant of the persistent Euler kernel.
//
// Same tile / slot / sliced-ELL design as k_resident (oscb_resident.cuh, read that header
// first), specialised for the throughput mode so that the per-oscillator work -- which costs
// as many instructions as a degree-20 gather -- is as lean as the gather itself:
//
//   * every shared-memory access uses a 32-bit shared address held in a register (row table,
//     (cos, sin) pairs, phases); the row table is one u32 per own row (row*RT | G << 16) read
//     through a running pointer, so there is no index arithmetic per row;
//   * phases live in shared memory next to the pairs when they fit (PHI_SMEM), else in the
//     tile's L2-resident slab;
//   * N = 2 (OIM / max-cut, NMODE == 2): the SHIL harmonic is 2 s c, and scoring costs one
//     LEA.HI per gather on the step AFTER a scored step: with c_j = cospi(2 phi_j) already in
//     a register, [c_j < 0] IS the lattice state of j (0.25 < phi < 0.75, dynamics.py:203-213;
//     pass B canonicalises -0 to +0, and tests/ check the equivalence over every float in
//     [0, 1)).  A row contributes deg - neg or neg differing neighbours depending on its own
//     state; the tile sum is twice the cut.  Trace samples and the first/last state still go
//     through the explicit scoring pass;
//   * other N (NMODE == 0): lattice states as bytes in shared memory, explicit scoring pass;
//   * Box-Muller on the MUFU unit (lg2 / sin / cos / sqrt approximations, |err| ~ 1e-6 on a
//     unit normal), noise off is a uniform branch.
//
// Arithmetic of a step (float32, FMA-contracted; parity is by tolerance / distribution):
//   sum = sum_j w_ij (c_j, s_j)            packed FADD2 / FFMA2
//   acc = s_i sum.x - c_i sum.y            == sum_j w_ij sin(2pi(phi_i - phi_j))   (dynamics.py:170)
//   x   = phi + hK acc - h ks shil + kn sqrt(h) xi ;  phi' = x - floor(x)           (dynamics.py:171-172)
#pragma once
#include "oscb_resident.cuh"

namespace oscb {

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ float lds_f32(uint32_t addr)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v)
{
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_pair(uint32_t addr, float c, float s)
{
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(c), "f"(s) : "memory");
}
__device__ __forceinline__ uint2 lds_u64(uint32_t addr)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t addr)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
    return v;
}

// four standard normals from one Philox block, MUFU Box-Muller (same draw -> same normal as
// normals4(float) up to ~1e-6)
__device__ __forceinline__ void normals4_fast(uint4 x, float &z0, float &z1, float &z2, float &z3)
{
    const float inv32 = 2.3283064365386963e-10f;
    const float u0 = fminf(fmaf((float)x.x, inv32, 0.5f * inv32), 1.0f);
    const float u1 = fminf(fmaf((float)x.z, inv32, 0.5f * inv32), 1.0f);
    float r0, r1;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(-1.3862943611198906f * __log2f(u0)));
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(-1.3862943611198906f * __log2f(u1)));
    // angle 2 pi v, v in [0, 1): fold to [-pi, pi) first, where the MUFU approximations are tightest
    const float v0 = (float)x.y * inv32, v1 = (float)x.w * inv32;
    const float a0 = 6.283185307179586f * (v0 - (v0 >= 0.5f ? 1.0f : 0.0f));
    const float a1 = 6.283185307179586f * (v1 - (v1 >= 0.5f ? 1.0f : 0.0f));
    z0 = r0 * __cosf(a0); z1 = r0 * __sinf(a0);
    z2 = r1 * __cosf(a1); z3 = r1 * __sinf(a1);
}

// Everything the kernel needs, precomputed on the host so that the hot loops read constants
// straight from the parameter bank instead of re-deriving them under register pressure.
struct FastArgs {
    int n, nRT, RT, LRT, C, W, n_rows /* 4 * rounds */, R_real;
    int n_group_rows;
    int piggy;                         // N = 2, unit weights, max-cut: score during the next gather
    int deg_smem;                      // the degree table of the piggyback is staged in shared memory
    uint32_t off_cs, off_phi, off_st, off_rows, off_g, off_deg, off_part, off_misc, off_stream, off_w, smem_total;
    float hK, knsh;
    double h, ks_max, ks_period, ks_scale /* h (x2 for N = 2) */;
    TrigConst tc;
    int noise_on, maximize, use_target, initial_sample, n_sample_steps, sample_offset;
    long long step_begin, step_end, cadence, trace_stride;
    double target;
    const int *warp_start;             // [W]
    const uint16_t *rows;              // [W * n_rows * C] own row * RT (>= nRT: none)
    const uint32_t *ginfo;             // [W * rounds]
    const uint16_t *deg;               // [W * n_rows * C]
    const uint2 *stream;               // [(n_group_rows + 1) * C]
    const float *wstream;              // [(n_group_rows + 1) * C * 4]
    float *phi;                        // [tiles][n][RT]
    const uint64_t *seeds;
    const long long *sample_steps;
    double *best_obj, *energy, *best_trace;
    uint8_t *best_states;
    long long *first_hit;
    unsigned long long *nonfinite;
};

// shared-memory layout of the float32 kernel; filled into FastArgs by the host
// Self-test of the N = 2 scoring shortcut: for EVERY float32 phase p in [0, 1) the sign bit of
// cospi(2p) + 0 (what pass B stores) must equal the reference threshold of p (dynamics.py:203-213).
__global__ void k_selftest_sign_state(unsigned long long *mismatches)
{
    const unsigned long long total = 0x3F800000ull;            // bit patterns of [0, 1)
    unsigned long long bad = 0;
    for (unsigned long long q = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (unsigned long long)gridDim.x * blockDim.x) {
        const float p = __uint_as_float((uint32_t)q);
        float s, co;
        sincospif(2.0f * p, &s, &co);
        const uint32_t by_sign = __float_as_uint(co + 0.0f) >> 31;
        if (by_sign != (uint32_t)threshold_state((double)p, 2)) ++bad;
    }
    if (bad) atomicAdd(mismatches, bad);
}

struct FastSmem {
    size_t cs, phi, st, rows, g, deg, part, misc, stream, wstream, total;
    __host__ static FastSmem make(int n, int RT, int C, int T, int W, int n_group_rows, bool need_states, bool need_deg,
                                  bool phi_smem, bool idx_smem, bool weighted)
    {
        FastSmem s;
        size_t o = 0;
        auto take = [&](size_t bytes) { size_t at = o; o += (bytes + 15) & ~(size_t)15; return at; };
        s.cs = take((size_t)(n + OSCB_PAD_ROWS) * RT * 8);
        s.phi = take(phi_smem ? (size_t)n * RT * 4 : 0);
        s.st = take(need_states ? (size_t)(n + OSCB_PAD_ROWS) * RT : 0);
        s.rows = take((size_t)W * T * 4 * C * 2);
        s.g = take((size_t)W * T * 4);
        s.deg = take(need_deg ? (size_t)W * T * 4 * C * 2 : 0);
        s.part = take((size_t)W * RT * 8);
        s.misc = take((size_t)RT * 16 + 32);
        s.stream = take(idx_smem ? (size_t)(n_group_rows + 1) * C * 8 : 0);
        s.wstream = take(idx_smem && weighted ? (size_t)(n_group_rows + 1) * C * 16 : 0);
        s.total = o;
        return s;
    }
};

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u8(uint32_t addr, uint32_t v)
{
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// NMODE: 2 = two lattice states (state = sign of the cosine); 0 = any N, state bytes.
template <int NMODE, bool WEIGHTED, bool IDX_SMEM, bool PHI_SMEM>
__global__ void __launch_bounds__(1024, 1) k_resident_fast(const FastArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, NT = blockDim.x;
    const uint32_t smem32 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const int lane = tid & 31, warp = tid >> 5;
    const int r = lane & (a.RT - 1), c = lane >> a.LRT;
    const int tile = blockIdx.x;
    const int rg = tile * a.RT + r;
    const bool live = rg < a.R_real;
    float *phi_g = a.phi + (size_t)tile * a.nRT + r;                        // the tile's slab (global), + row*RT

    // lane-resident shared addresses (+ row*RT scaled by the element size)
    const uint32_t cs32 = smem32 + a.off_cs + r * 8;
    const uint32_t phi32 = smem32 + a.off_phi + r * 4;
    const uint32_t st32 = smem32 + a.off_st + r;
    const uint32_t rows32 = smem32 + a.off_rows + ((warp * a.n_rows) * a.C + c) * 2;   // own rows, stride C*2
    const uint32_t g32 = smem32 + a.off_g + warp * a.n_rows;                           // G per row position
    const uint16_t *deg_lane = (a.deg_smem ? reinterpret_cast<const uint16_t *>(smem_raw + a.off_deg) : a.deg) + (warp * a.n_rows) * a.C + c;
    double *part = reinterpret_cast<double *>(smem_raw + a.off_part);
    double *best_s = reinterpret_cast<double *>(smem_raw + a.off_misc);
    int *improved_s = reinterpret_cast<int *>(smem_raw + a.off_misc + a.RT * 8);
    float *ks_s = reinterpret_cast<float *>(smem_raw + a.off_misc + a.RT * 16);        // [2]: ks_scale * ks(step)

    // ---- prologue -------------------------------------------------------------------------------
    {
        uint16_t *rows = reinterpret_cast<uint16_t *>(smem_raw + a.off_rows);
        uint8_t *gs = smem_raw + a.off_g;
        uint16_t *degs = reinterpret_cast<uint16_t *>(smem_raw + a.off_deg);
        const int total_rows = a.W * a.n_rows;
        for (int q = tid; q < total_rows * a.C; q += NT) {
            rows[q] = a.rows[q];
            if (a.deg_smem) degs[q] = a.deg[q];
        }
        for (int q = tid; q < total_rows; q += NT) gs[q] = (uint8_t)((a.ginfo[q >> 2] >> (8 * (q & 3))) & 0xFFu);
        if (IDX_SMEM) {
            uint2 *dst = reinterpret_cast<uint2 *>(smem_raw + a.off_stream);
            for (int q = tid; q < (a.n_group_rows + 1) * a.C; q += NT) dst[q] = a.stream[q];
            if (WEIGHTED) {
                float *wd = reinterpret_cast<float *>(smem_raw + a.off_w);
                for (int q = tid; q < (a.n_group_rows + 1) * a.C * 4; q += NT) wd[q] = a.wstream[q];
            }
        }
        float2 *cs = reinterpret_cast<float2 *>(smem_raw + a.off_cs);
        float *phis = reinterpret_cast<float *>(smem_raw + a.off_phi);
        const float *slab = a.phi + (size_t)tile * a.nRT;
        for (int q = tid; q < a.nRT; q += NT) {
            const float p = slab[q];
            float s, co;
            sincospif(2.0f * p, &s, &co);
            cs[q] = make_float2(co + 0.0f, s);
            if (PHI_SMEM) phis[q] = p;
        }
        for (int q = tid; q < OSCB_PAD_ROWS * a.RT; q += NT) {
            cs[a.nRT + q] = make_float2(0.0f, 0.0f);
            if (NMODE != 2) (smem_raw + a.off_st)[a.nRT + q] = 255;
        }
        if (tid < a.RT) {
            best_s[tid] = a.best_obj[tile * a.RT + tid];
            improved_s[tid] = 0;
        }
        if (tid == 0) ks_s[a.step_begin & 1] = (float)(a.ks_scale * ks_value(a.ks_max, a.ks_period, (double)a.step_begin * a.h));
    }
    const uint64_t seed = a.seeds[rg];
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const int gp0 = a.warp_start[warp];
    const uint2 *stream_g = a.stream + (size_t)gp0 * a.C + c;               // this lane's slot, stride C
    const uint32_t stream32 = smem32 + a.off_stream + (uint32_t)(gp0 * a.C + c) * 8;
    const float *w_g = a.wstream + ((size_t)gp0 * a.C + c) * 4;
    const uint32_t w32 = smem32 + a.off_w + (uint32_t)(gp0 * a.C + c) * 16;
    __syncthreads();

    auto load_phi = [&](uint32_t iRT) -> float { return PHI_SMEM ? lds_f32(phi32 + iRT * 4) : phi_g[iRT]; };
    auto store_phi = [&](uint32_t iRT, float v) {
        if (PHI_SMEM) sts_f32(phi32 + iRT * 4, v);
        else phi_g[iRT] = v;
    };
    auto pair_at = [&](uint32_t idRT) -> float2 { float2 v; lds_pair(pair_addr<3>(idRT, cs32), v); return v; };
    auto group_at = [&](int g) -> uint2 { return IDX_SMEM ? lds_u64(stream32 + (uint32_t)(g * a.C) * 8) : stream_g[g * a.C]; };
    auto weights_at = [&](int g) -> float4 {
        return IDX_SMEM ? lds_f4(w32 + (uint32_t)(g * a.C) * 16) : *reinterpret_cast<const float4 *>(w_g + (size_t)(g * a.C) * 4);
    };
    auto row_at = [&](int row) -> uint32_t { return lds_u16(rows32 + (uint32_t)(row * a.C) * 2); };
    auto state_of = [&](uint32_t idRT) -> uint32_t {
        if (NMODE == 2) return __float_as_uint(pair_at(idRT).x) >> 31;
        return lds_u8(st32 + idRT);
    };

    // explicit scoring pass over the state in cs (/ state bytes); sample_col >= 0 also records the trace column
    auto score_current = [&](long long step_label, int sample_col) {
        double obj_part = 0.0, en_part = 0.0;
        int g = 0;
        for (int row = 0; row < a.n_rows; ++row) {
            const uint32_t iRT = row_at(row);
            const int G = (int)lds_u8(g32 + row);
            if (iRT < (uint32_t)a.nRT) {
                const uint32_t si = state_of(iRT);
                const float2 own = pair_at(iRT);
                int count = 0;
                double wsum = 0.0;
                for (int gg = 0; gg < G; ++gg) {
                    const uint2 pk = group_at(g + gg);
                    float4 w4 = make_float4(1.f, 1.f, 1.f, 1.f);
                    if (WEIGHTED) w4 = weights_at(g + gg);
                    const uint32_t jj[4] = {pk.x & 0xffffu, pk.x >> 16, pk.y & 0xffffu, pk.y >> 16};
                    const float ww[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t jRT = jj[u];
                        if (jRT > iRT && jRT < (uint32_t)a.nRT) {          // canonical pairs i < j only
                            const bool same = state_of(jRT) == si;
                            const bool hit = a.maximize ? !same : same;
                            if (WEIGHTED) { if (hit) wsum += a.maximize ? (double)ww[u] : 1.0; }
                            else count += hit ? 1 : 0;
                            if (sample_col >= 0) {
                                const float2 v = pair_at(jRT);
                                en_part += (double)ww[u] * ((double)own.x * (double)v.x + (double)own.y * (double)v.y);
                            }
                        }
                    }
                }
                obj_part += WEIGHTED ? wsum : (double)count;
            }
            g += G;
        }
        const double obj = tile_reduce(obj_part, a.RT, part, tid, a.W);
        if (tid < a.RT) {
            const double b = best_s[tid];
            const bool better = a.maximize ? (obj > b) : (obj < b);
            improved_s[tid] = better ? 1 : 0;
            if (better) {
                best_s[tid] = obj;
                const int gi = tile * a.RT + tid;
                if (a.use_target && a.first_hit[gi] < 0 && (a.maximize ? (obj >= a.target) : (obj <= a.target)))
                    a.first_hit[gi] = step_label;
            }
        }
        __syncthreads();
        if (improved_s[r] && live) {
            uint8_t *dst = a.best_states + (size_t)rg * a.n;
            for (int row = 0; row < a.n_rows; ++row) {
                const uint32_t iRT = row_at(row);
                if (iRT < (uint32_t)a.nRT) dst[iRT >> a.LRT] = (uint8_t)state_of(iRT);
            }
        }
        if (sample_col >= 0) {
            const double en = tile_reduce(en_part, a.RT, part, tid, a.W);
            if (tid < a.RT) {
                const size_t gi = (size_t)(tile * a.RT + tid);
                a.energy[gi * a.trace_stride + sample_col] = en;
                a.best_trace[gi * a.trace_stride + sample_col] = best_s[tid];
            }
        }
        __syncthreads();
    };

    // N = 2: `twice_cut` was counted during the gather of step `step_label + 1`
    auto finish_piggyback = [&](int twice_cut, long long step_label) {
        const double obj = 0.5 * tile_reduce((double)twice_cut, a.RT, part, tid, a.W);
        if (tid < a.RT) {
            const double b = best_s[tid];
            const bool better = obj > b;
            improved_s[tid] = better ? 1 : 0;
            if (better) {
                best_s[tid] = obj;
                const int gi = tile * a.RT + tid;
                if (a.use_target && a.first_hit[gi] < 0 && obj >= a.target) a.first_hit[gi] = step_label;
            }
        }
        __syncthreads();
        if (improved_s[r] && live) {               // cs still holds the scored state (pass B comes later)
            uint8_t *dst = a.best_states + (size_t)rg * a.n;
            for (int row = 0; row < a.n_rows; ++row) {
                const uint32_t iRT = row_at(row);
                if (iRT < (uint32_t)a.nRT) dst[iRT >> a.LRT] = (uint8_t)(__float_as_uint(pair_at(iRT).x) >> 31);
            }
        }
    };

    int sample_cur = 0;
    while (sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] < a.step_begin) ++sample_cur;

    if (a.initial_sample) {
        if (NMODE != 2) {
            for (int row = 0; row < a.n_rows; ++row) {
                const uint32_t iRT = row_at(row);
                if (iRT < (uint32_t)a.nRT) sts_u8(st32 + iRT, (uint32_t)threshold_state((double)load_phi(iRT), a.tc.n_states));
            }
            __syncthreads();
        }
        score_current(-1, 0);
    }

    bool pending = false;        // N = 2: the state after the previous step still has to be scored
    long long pending_label = 0;

    // ---- time loop ------------------------------------------------------------------------------
#pragma unroll 1
    for (long long step = a.step_begin; step < a.step_end; ++step) {
        const float hks = ks_s[step & 1];           // h*ks, or 2*h*ks for N = 2
        const bool is_sample = sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] == step;
        const bool cadence_hit = a.cadence > 0 && step % a.cadence == 0;
        const bool count_now = NMODE == 2 && !WEIGHTED && pending;
        int twice_cut = 0;

        // pass A ------------------------------------------------------------------------------
        // The stream of a warp is contiguous: a running pointer walks it and the next group is
        // always loaded one group ahead of its use (the pad row covers the last one).
        uint32_t sp32 = stream32, wp32 = w32;
        const uint2 *spg = stream_g;
        const float *wpg = w_g;
        auto next_group = [&]() -> uint2 {
            if (IDX_SMEM) { sp32 += (uint32_t)a.C * 8; return lds_u64(sp32); }
            spg += a.C;
            return *spg;
        };
        auto next_weights = [&]() -> float4 {       // weights of the group consumed now, then advance
            float4 w4;
            if (IDX_SMEM) { w4 = lds_f4(wp32); wp32 += (uint32_t)a.C * 16; }
            else { w4 = *reinterpret_cast<const float4 *>(wpg); wpg += a.C * 4; }
            return w4;
        };
        uint2 pk = IDX_SMEM ? lds_u64(sp32) : *spg;
        float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
#pragma unroll 1
        for (int row = 0; row < a.n_rows; ++row) {
            const uint32_t iRT = row_at(row);
            const int G = (int)lds_u8(g32 + row);
            const bool valid = iRT < (uint32_t)a.nRT;
            const float p = load_phi(iRT);              // issued a whole gather ahead of its use
            if ((row & 3) == 0 && a.noise_on && valid)
                normals4_fast(philox4x32_10(make_uint4((iRT >> a.LRT) >> 2, (uint32_t)step, (uint32_t)(step >> 32), 0x6F736362u), key),
                              z0, z1, z2, z3);
            float2 sum = make_float2(0.f, 0.f);
            int neg = 0;
            if (NMODE == 2 && !WEIGHTED && count_now) {
                // scoring step: the sign bit of every gathered cosine is the neighbour's lattice state
#pragma unroll 2
                for (int gg = 0; gg < G; ++gg) {
                    const uint2 nx = next_group();
                    const float2 v0 = pair_at(pk.x & 0xffffu), v1 = pair_at(pk.x >> 16);
                    const float2 v2 = pair_at(pk.y & 0xffffu), v3 = pair_at(pk.y >> 16);
                    sum = __fadd2_rn(sum, __fadd2_rn(__fadd2_rn(v0, v1), __fadd2_rn(v2, v3)));
                    neg += (int)(__float_as_uint(v0.x) >> 31) + (int)(__float_as_uint(v1.x) >> 31);
                    neg += (int)(__float_as_uint(v2.x) >> 31) + (int)(__float_as_uint(v3.x) >> 31);
                    pk = nx;
                }
            } else {
#pragma unroll 2
                for (int gg = 0; gg < G; ++gg) {
                    const uint2 nx = next_group();
                    const float2 v0 = pair_at(pk.x & 0xffffu), v1 = pair_at(pk.x >> 16);
                    const float2 v2 = pair_at(pk.y & 0xffffu), v3 = pair_at(pk.y >> 16);
                    if (WEIGHTED) {
                        const float4 w4 = next_weights();
                        sum = __ffma2_rn(make_float2(w4.x, w4.x), v0, sum);
                        sum = __ffma2_rn(make_float2(w4.y, w4.y), v1, sum);
                        sum = __ffma2_rn(make_float2(w4.z, w4.z), v2, sum);
                        sum = __ffma2_rn(make_float2(w4.w, w4.w), v3, sum);
                    } else {
                        sum = __fadd2_rn(sum, __fadd2_rn(__fadd2_rn(v0, v1), __fadd2_rn(v2, v3)));
                    }
                    pk = nx;
                }
            }
            if (valid) {
                const float2 own = pair_at(iRT);
                const float ci = own.x, si = own.y;
                if (NMODE == 2 && !WEIGHTED && count_now)   // differing neighbours: deg - neg if the row itself is in state 1
                    twice_cut += (ci < 0.f) ? (int)deg_lane[row * a.C] - neg : neg;
                const float acc = si * sum.x - ci * sum.y;
                float shil;
                if (NMODE == 2) shil = si * ci;                                  // hks holds 2 h ks
                else shil = shil_term(p, si, ci, a.tc);
                const uint32_t k = (iRT >> a.LRT) & 3u;
                const float kick = (k & 2u) ? ((k & 1u) ? z3 : z2) : ((k & 1u) ? z1 : z0);
                const float x = fmaf(a.hK, acc, fmaf(-hks, shil, fmaf(a.knsh, kick, p)));
                float y = x - floorf(x);
                y = (y >= 1.0f) ? 0.0f : y;
                if (!(fabsf(x) < INFINITY) && live) flag_nonfinite(a.nonfinite, (uint64_t)step, (uint32_t)rg, iRT >> a.LRT);
                store_phi(iRT, y);
            }
        }
        if (tid == 0) ks_s[(step + 1) & 1] = (float)(a.ks_scale * ks_value(a.ks_max, a.ks_period, (double)(step + 1) * a.h));
        if (count_now) {
            finish_piggyback(twice_cut, pending_label);
            pending = false;
        }
        __syncthreads();

        // pass B: pairs (and state bytes) of the new phases -------------------------------------
        const bool score_after = is_sample || cadence_hit;
#pragma unroll 1
        for (int row = 0; row < a.n_rows; ++row) {
            const uint32_t iRT = row_at(row);
            if (iRT < (uint32_t)a.nRT) {
                const float p = load_phi(iRT);
                float s, co;
                sincospif(2.0f * p, &s, &co);
                sts_pair(pair_addr<3>(iRT, cs32), co + 0.0f, s);
                if (NMODE != 2 && score_after) sts_u8(st32 + iRT, (uint32_t)threshold_state((double)p, a.tc.n_states));
            }
        }
        __syncthreads();

        if (is_sample) {
            score_current(step, a.sample_offset + sample_cur);
            ++sample_cur;
        } else if (cadence_hit) {
            if (NMODE == 2 && !WEIGHTED && a.piggy && step + 1 < a.step_end) {
                pending = true;
                pending_label = step;
            } else {
                score_current(step, -1);
            }
        }
    }
    if (tid < a.RT) a.best_obj[tile * a.RT + tid] = best_s[tid];
    if (!PHI_SMEM) return;
    __syncthreads();
    {
        const float *phis = reinterpret_cast<const float *>(smem_raw + a.off_phi);
        float *slab = a.phi + (size_t)tile * a.nRT;
        for (int q = tid; q < a.nRT; q += NT) slab[q] = phis[q];
    }
}

} // namespace oscb
