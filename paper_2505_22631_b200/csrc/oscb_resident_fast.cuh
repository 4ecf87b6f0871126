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
//     a register, its SIGN BIT is the lattice state of j (0.25 < phi < 0.75, dynamics.py:203-213;
//     trig_turns_direct sets the bit from that exact comparison, and oscb_selftest_sign_state checks
//     it over every float in [0, 1)).  A row contributes deg - neg or neg differing neighbours depending on its own
//     state; the tile sum is twice the cut.  Trace samples and the first/last state still go
//     through the explicit scoring pass;
//   * other N (NMODE == 0): lattice states as bytes in shared memory, explicit scoring pass;
//   * RPL replicas per lane (1 or 2): with RPL = 2 a lane owns two adjacent replicas, so one
//     LDS.128 fetches both (cos, sin) pairs of a neighbour and the index unpacking / address
//     arithmetic of a gather is shared by two updates;
//   * Box-Muller on the MUFU unit (lg2 / sin / cos / sqrt approximations, |err| ~ 1e-6 on a
//     unit normal), noise off is a uniform branch.
//
// Arithmetic of a step (float32, FMA-contracted; parity is by tolerance / distribution):
//   sum = sum_j w_ij (c_j, s_j)            packed FADD2 / FFMA2
//   acc = s_i sum.x - c_i sum.y            == sum_j w_ij sin(2pi(phi_i - phi_j))   (dynamics.py:170)
//   x   = phi + hK acc - h ks shil + kn sqrt(h) xi ;  phi' = x - floor(x)           (dynamics.py:171-172)
#pragma once
#include "oscb_resident.cuh"
#include "oscb_fastmath.cuh"
#include <string.h>

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

// Everything the kernel needs, precomputed on the host so that the hot loops read constants
// straight from the parameter bank instead of re-deriving them under register pressure.
struct FastArgs {
    int n, nRT, RT, LRT, LPS, LLPS /* lanes per slot = RT / RPL and its log2 */, C, W, n_rows /* 4 * rounds */, R_real;
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
    const uint16_t *deg;               // [W * n_rows * C]  row degrees (unit weights)
    const float *rowsum;               // [W * n_rows * C]  row weight sums (integer-valued weights)
    const uint2 *stream;               // [(n_group_rows + 1) * C]
    const float *wstream;              // [(n_group_rows + 1) * C * 4]
    float *phi;                        // [tiles][n][RT] (+ one padding row at the very end)
    float2 *cs_next;                   // [tiles][n][RT] next-step (cos, sin) pairs, L2-resident staging (N = 2 kernels)
    const uint64_t *seeds;
    const long long *sample_steps;
    const float *hks_table;            // [step_end - step_begin + 1]  ks_scale * ks(step), computed on the host in float64
    int n_bnd;                         // > 0: lattice states from float32 decision boundaries (N <= 8), else the float64 rule
    float bnd[8];                      // bnd[k] = smallest float32 phase whose reference state is (k + 1) % N
    double *best_obj, *energy, *best_trace;
    uint8_t *best_states;
    long long *first_hit;
    unsigned long long *nonfinite;
};

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
        trig_turns_direct(p, s, co);
        const uint32_t by_sign = __float_as_uint(co) >> 31;
        if (by_sign != (uint32_t)threshold_state((double)p, 2)) ++bad;
        // and the values themselves stay within the MUFU error of the exact ones
        float s_ref, c_ref;
        sincospif(2.0f * p, &s_ref, &c_ref);
        if (!(fabsf(s - s_ref) <= 2e-6f && fabsf(co - c_ref) <= 2e-6f)) ++bad;
    }
    if (bad) atomicAdd(mismatches, bad);
}

// Self-test of the boundary table for N states: every float32 phase in [0, 1) must get the state of
// the float64 reference rule.
__global__ void k_selftest_boundaries(int n_states, FastArgs a, unsigned long long *mismatches)
{
    const unsigned long long total = 0x3F800000ull;
    unsigned long long bad = 0;
    for (unsigned long long q = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (unsigned long long)gridDim.x * blockDim.x) {
        const float p = __uint_as_float((uint32_t)q);
        if (state_from_boundaries(p, a.bnd, a.n_bnd) != (uint32_t)threshold_state((double)p, n_states)) ++bad;
    }
    if (bad) atomicAdd(mismatches, bad);
}

// shared-memory layout of the float32 kernel; filled into FastArgs by the host
struct FastSmem {
    size_t cs, phi, st, rows, g, deg, part, misc, stream, wstream, total;
    __host__ static FastSmem make(int n, int RT, int C, int T, int W, int n_group_rows, bool need_states, bool need_deg,
                                  bool phi_smem, bool idx_smem, bool weighted)
    {
        FastSmem s;
        size_t o = 0;
        auto take = [&](size_t bytes) { size_t at = o; o += (bytes + 15) & ~(size_t)15; return at; };
        s.cs = take((size_t)(n + OSCB_PAD_ROWS) * RT * 8);
        s.phi = take(phi_smem ? (size_t)(n + 1) * RT * 4 : 0);
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
__device__ __forceinline__ float2 lds_f2(uint32_t addr)
{
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
    return v;
}

// (cos, sin) pairs of RPL adjacent replicas of one row: one LDS.64 or one LDS.128
template <int RPL> struct PairPack;
template <> struct PairPack<1> {
    float2 v[1];
    __device__ __forceinline__ void load(uint32_t addr) { v[0] = lds_f2(addr); }
};
template <> struct PairPack<2> {
    float2 v[2];
    __device__ __forceinline__ void load(uint32_t addr)
    {
        const float4 t = lds_f4(addr);
        v[0] = make_float2(t.x, t.y);
        v[1] = make_float2(t.z, t.w);
    }
};

// Sum RPL per-lane values over all lanes of the CTA that hold the same replicas (same lane-in-slot
// q), in a fixed order.  Replica q*RPL + e ends up in part2[...]; result for replica `tid` valid
// in threads tid < RT.  Two barriers inside.
template <int RPL>
__device__ __forceinline__ double tile_reduce_rpl(const double (&v)[RPL], int RT, int LPS, double *part, int tid, int nwarps)
{
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
        double x = v[e];
        for (int off = 16; off >= LPS; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        if (lane < LPS) part[warp * RT + lane * RPL + e] = x;
    }
    __syncthreads();
    double tot = 0.0;
    if (tid < RT)
        for (int w = 0; w < nwarps; ++w) tot += part[w * RT + tid];
    __syncthreads();
    return tot;
}

// NMODE: 2 = two lattice states (state = sign of the cosine); 0 = any N, state bytes.
// RPL:   replicas per lane.
template <int NMODE, bool WEIGHTED, bool IDX_SMEM, bool PHI_SMEM, int RPL>
__global__ void __launch_bounds__(1024, 1) k_resident_fast(const FastArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool PIGGY = true;          // N = 2 max-cut (sign bits) and N-state colouring (state bytes): score during the next gather
    const int tid = threadIdx.x, NT = blockDim.x;
    const uint32_t smem32 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const int lane = tid & 31, warp = tid >> 5;
    const int q = lane & (a.LPS - 1), c = lane >> a.LLPS;
    const int r0 = q * RPL;                                 // first replica (inside the tile) of this lane
    const int tile = blockIdx.x;
    const int rg0 = tile * a.RT + r0;
    float *phi_g = a.phi + (size_t)tile * a.nRT + r0;       // the tile's slab (global), + row*RT
    float2 *stage_g = a.cs_next + (size_t)tile * a.nRT + r0; // next-step pairs of this lane's replicas, + row*RT
    // N = 2: the trig of the new phase is done right in the row epilogue of pass A (where it overlaps
    // other warps' gathers) and parked in an L2-resident staging slab; pass B is then a plain copy.
    constexpr bool STAGED = NMODE == 2;

    // lane-resident shared addresses (+ row*RT scaled by the element size)
    const uint32_t cs32 = smem32 + a.off_cs + r0 * 8;
    const uint32_t phi32 = smem32 + a.off_phi + r0 * 4;
    const uint32_t st32 = smem32 + a.off_st + r0;
    const uint32_t rows32 = smem32 + a.off_rows + ((warp * a.n_rows) * a.C + c) * 2;   // own rows, stride C*2
    const uint32_t g32 = smem32 + a.off_g + warp * a.n_rows;                           // G per row position
    const uint16_t *deg_lane = (a.deg_smem ? reinterpret_cast<const uint16_t *>(smem_raw + a.off_deg) : a.deg) + (warp * a.n_rows) * a.C + c;
    const float *rowsum_lane = a.rowsum + (warp * a.n_rows) * a.C + c;
    double *part = reinterpret_cast<double *>(smem_raw + a.off_part);
    double *best_s = reinterpret_cast<double *>(smem_raw + a.off_misc);
    int *improved_s = reinterpret_cast<int *>(smem_raw + a.off_misc + a.RT * 8);

    // ---- prologue -------------------------------------------------------------------------------
    {
        uint16_t *rows = reinterpret_cast<uint16_t *>(smem_raw + a.off_rows);
        uint8_t *gs = smem_raw + a.off_g;
        uint16_t *degs = reinterpret_cast<uint16_t *>(smem_raw + a.off_deg);
        const int total_rows = a.W * a.n_rows;
        for (int i = tid; i < total_rows * a.C; i += NT) {
            rows[i] = a.rows[i];
            if (a.deg_smem) degs[i] = a.deg[i];
        }
        for (int i = tid; i < total_rows; i += NT) gs[i] = (uint8_t)((a.ginfo[i >> 2] >> (8 * (i & 3))) & 0xFFu);
        if (IDX_SMEM) {
            uint2 *dst = reinterpret_cast<uint2 *>(smem_raw + a.off_stream);
            for (int i = tid; i < (a.n_group_rows + 1) * a.C; i += NT) dst[i] = a.stream[i];
            if (WEIGHTED) {
                float *wd = reinterpret_cast<float *>(smem_raw + a.off_w);
                for (int i = tid; i < (a.n_group_rows + 1) * a.C * 4; i += NT) wd[i] = a.wstream[i];
            }
        }
        float2 *cs = reinterpret_cast<float2 *>(smem_raw + a.off_cs);
        float *phis = reinterpret_cast<float *>(smem_raw + a.off_phi);
        const float *slab = a.phi + (size_t)tile * a.nRT;
        for (int i = tid; i < a.nRT; i += NT) {
            const float p = slab[i];
            float s, co;
            trig_turns_direct(p, s, co);
            cs[i] = make_float2(co, s);
            if (PHI_SMEM) phis[i] = p;
        }
        for (int i = tid; i < OSCB_PAD_ROWS * a.RT; i += NT) {
            cs[a.nRT + i] = make_float2(0.0f, 0.0f);
            if (NMODE != 2) (smem_raw + a.off_st)[a.nRT + i] = 255;
        }
        if (PHI_SMEM && tid < a.RT) phis[a.nRT + tid] = 0.0f;   // the row invalid slots load
        if (tid < a.RT) {
            best_s[tid] = a.best_obj[tile * a.RT + tid];
            improved_s[tid] = 0;
        }
    }
    uint2 key[RPL];
    bool live[RPL];
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
        const uint64_t seed = a.seeds[rg0 + e];
        key[e] = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
        live[e] = rg0 + e < a.R_real;
    }
    const int gp0 = a.warp_start[warp];
    const uint2 *stream_g = a.stream + (size_t)gp0 * a.C + c;               // this lane's slot, stride C
    const uint32_t stream32 = smem32 + a.off_stream + (uint32_t)(gp0 * a.C + c) * 8;
    const float *w_g = a.wstream + ((size_t)gp0 * a.C + c) * 4;
    const uint32_t w32 = smem32 + a.off_w + (uint32_t)(gp0 * a.C + c) * 16;
    __syncthreads();

    auto state_of_phase = [&](float p) -> uint32_t {
        return a.n_bnd > 0 ? state_from_boundaries(p, a.bnd, a.n_bnd) : (uint32_t)threshold_state((double)p, a.tc.n_states);
    };
    auto load_phi = [&](uint32_t iRT, float (&p)[RPL]) {
        if (RPL == 2) {
            float2 t;
            if (PHI_SMEM) t = lds_f2(phi32 + iRT * 4);
            else t = *reinterpret_cast<const float2 *>(phi_g + iRT);
            p[0] = t.x; p[RPL - 1] = t.y;
        } else {
            p[0] = PHI_SMEM ? lds_f32(phi32 + iRT * 4) : phi_g[iRT];
        }
    };
    auto store_phi = [&](uint32_t iRT, const float (&p)[RPL]) {
        if (RPL == 2) {
            if (PHI_SMEM) sts_pair(phi32 + iRT * 4, p[0], p[RPL - 1]);
            else *reinterpret_cast<float2 *>(phi_g + iRT) = make_float2(p[0], p[RPL - 1]);
        } else {
            if (PHI_SMEM) sts_f32(phi32 + iRT * 4, p[0]);
            else phi_g[iRT] = p[0];
        }
    };
    auto pairs_at = [&](uint32_t idRT) -> PairPack<RPL> { PairPack<RPL> pp; pp.load(pair_addr<3>(idRT, cs32)); return pp; };
    auto group_at = [&](int g) -> uint2 { return IDX_SMEM ? lds_u64(stream32 + (uint32_t)(g * a.C) * 8) : stream_g[g * a.C]; };
    auto weights_at = [&](int g) -> float4 {
        return IDX_SMEM ? lds_f4(w32 + (uint32_t)(g * a.C) * 16) : *reinterpret_cast<const float4 *>(w_g + (size_t)(g * a.C) * 4);
    };
    auto row_at = [&](int row) -> uint32_t { return lds_u16(rows32 + (uint32_t)(row * a.C) * 2); };
    auto states_of = [&](uint32_t idRT, uint32_t (&st)[RPL]) {
        if (NMODE == 2) {
            const PairPack<RPL> pp = pairs_at(idRT);
#pragma unroll
            for (int e = 0; e < RPL; ++e) st[e] = __float_as_uint(pp.v[e].x) >> 31;
        } else {
#pragma unroll
            for (int e = 0; e < RPL; ++e) st[e] = lds_u8(st32 + idRT + e);
        }
    };
    auto publish_states = [&]() {              // best_states rows of the replicas that just improved
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
            if (improved_s[r0 + e] && live[e]) {
                uint8_t *dst = a.best_states + (size_t)(rg0 + e) * a.n;
                for (int row = 0; row < a.n_rows; ++row) {
                    const uint32_t iRT = row_at(row);
                    if (iRT < (uint32_t)a.nRT) {
                        uint32_t st[RPL];
                        states_of(iRT, st);
                        dst[iRT >> a.LRT] = (uint8_t)st[e];
                    }
                }
            }
        }
    };
    auto record_best = [&](double obj, long long step_label) {     // threads tid < RT: strict improvement
        const double b = best_s[tid];
        const bool better = a.maximize ? (obj > b) : (obj < b);
        improved_s[tid] = better ? 1 : 0;
        if (better) {
            best_s[tid] = obj;
            const int gi = tile * a.RT + tid;
            if (a.use_target && a.first_hit[gi] < 0 && (a.maximize ? (obj >= a.target) : (obj <= a.target)))
                a.first_hit[gi] = step_label;
        }
    };

    // explicit scoring pass over the state in cs (/ state bytes); sample_col >= 0 also records the trace column
    auto score_current = [&](long long step_label, int sample_col) {
        double obj_part[RPL], en_part[RPL];
#pragma unroll
        for (int e = 0; e < RPL; ++e) { obj_part[e] = 0.0; en_part[e] = 0.0; }
        int g = 0;
        for (int row = 0; row < a.n_rows; ++row) {
            const uint32_t iRT = row_at(row);
            const int G = (int)lds_u8(g32 + row);
            if (iRT < (uint32_t)a.nRT) {
                uint32_t si[RPL];
                states_of(iRT, si);
                const PairPack<RPL> own = pairs_at(iRT);
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
                            uint32_t sj[RPL];
                            states_of(jRT, sj);
                            const PairPack<RPL> v = pairs_at(jRT);
#pragma unroll
                            for (int e = 0; e < RPL; ++e) {
                                const bool same = sj[e] == si[e];
                                const bool hit = a.maximize ? !same : same;
                                if (hit) obj_part[e] += (WEIGHTED && a.maximize) ? (double)ww[u] : 1.0;
                                if (sample_col >= 0)
                                    en_part[e] += (double)ww[u] * ((double)own.v[e].x * (double)v.v[e].x + (double)own.v[e].y * (double)v.v[e].y);
                            }
                        }
                    }
                }
            }
            g += G;
        }
        const double obj = tile_reduce_rpl<RPL>(obj_part, a.RT, a.LPS, part, tid, a.W);
        if (tid < a.RT) record_best(obj, step_label);
        __syncthreads();
        publish_states();
        if (sample_col >= 0) {
            const double en = tile_reduce_rpl<RPL>(en_part, a.RT, a.LPS, part, tid, a.W);
            if (tid < a.RT) {
                const size_t gi = (size_t)(tile * a.RT + tid);
                a.energy[gi * a.trace_stride + sample_col] = en;
                a.best_trace[gi * a.trace_stride + sample_col] = best_s[tid];
            }
        }
        __syncthreads();
    };

    int sample_cur = 0;
    while (sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] < a.step_begin) ++sample_cur;

    if (a.initial_sample) {
        if (NMODE != 2) {
            for (int row = 0; row < a.n_rows; ++row) {
                const uint32_t iRT = row_at(row);
                if (iRT < (uint32_t)a.nRT) {
                    float p[RPL];
                    load_phi(iRT, p);
#pragma unroll
                    for (int e = 0; e < RPL; ++e) sts_u8(st32 + iRT + e, state_of_phase(p[e]));
                }
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
        const float hks = __ldg(a.hks_table + (step - a.step_begin));   // h*ks, or 2*h*ks for N = 2 (host table: no float64 fmod here)
        const bool is_sample = sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] == step;
        const bool cadence_hit = a.cadence > 0 && step % a.cadence == 0;
        const bool count_now = PIGGY && pending;
        int twice_cut[RPL];            // unit weights: exact integer count
        float twice_cut_w[RPL];        // integer-valued weights: exact in float32 below 2^24
#pragma unroll
        for (int e = 0; e < RPL; ++e) { twice_cut[e] = 0; twice_cut_w[e] = 0.f; }

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
        float z[RPL][4];
#pragma unroll
        for (int e = 0; e < RPL; ++e) { z[e][0] = 0.f; z[e][1] = 0.f; z[e][2] = 0.f; z[e][3] = 0.f; }
#pragma unroll 1
        for (int row = 0; row < a.n_rows; ++row) {
            const uint32_t iRT = row_at(row);
            const int G = (int)lds_u8(g32 + row);
            const bool valid = iRT < (uint32_t)a.nRT;
            float p[RPL];
            load_phi(iRT, p);                           // issued a whole gather ahead of its use
            // One Philox block per quad and replica.  Even warps draw it before the quad's first
            // gather, odd warps after it, so that at any time half of the SM's warps are on the
            // ALU/MUFU pipes while the other half keep the shared-memory pipe busy.
            const bool draw = (row & 3) == 0 && a.noise_on && valid;
            auto draw_noise = [&]() {
#pragma unroll
                for (int e = 0; e < RPL; ++e)
                    normals4_fast(philox4x32_10(make_uint4((iRT >> a.LRT) >> 2, (uint32_t)step, (uint32_t)(step >> 32), 0x6F736362u), key[e]),
                                  z[e][0], z[e][1], z[e][2], z[e][3]);
            };
            if (draw && !(warp & 1)) draw_noise();
            float2 sum[RPL];
            int neg[RPL];
            float negw[RPL];
#pragma unroll
            for (int e = 0; e < RPL; ++e) { sum[e] = make_float2(0.f, 0.f); neg[e] = 0; negw[e] = 0.f; }
            if (PIGGY && count_now && NMODE != 2) {
                // colouring, scoring step: count the neighbours in the row's own state (state bytes of the
                // scored phases; padding rows hold 255 and never match)
                uint32_t own_st[RPL];
                states_of(iRT, own_st);
#pragma unroll 1
                for (int gg = 0; gg < G; ++gg) {
                    const uint2 nx = next_group();
                    const uint32_t j0 = pk.x & 0xffffu, j1 = pk.x >> 16, j2 = pk.y & 0xffffu, j3 = pk.y >> 16;
                    const PairPack<RPL> v0 = pairs_at(j0), v1 = pairs_at(j1), v2 = pairs_at(j2), v3 = pairs_at(j3);
                    uint32_t s0[RPL], s1[RPL], s2[RPL], s3[RPL];
                    states_of(j0, s0); states_of(j1, s1); states_of(j2, s2); states_of(j3, s3);
                    if (WEIGHTED) {
                        const float4 w4 = next_weights();
#pragma unroll
                        for (int e = 0; e < RPL; ++e) {              // same order as the non-scoring gather
                            sum[e] = __ffma2_rn(make_float2(w4.x, w4.x), v0.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.y, w4.y), v1.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.z, w4.z), v2.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.w, w4.w), v3.v[e], sum[e]);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < RPL; ++e)
                            sum[e] = __fadd2_rn(sum[e], __fadd2_rn(__fadd2_rn(v0.v[e], v1.v[e]), __fadd2_rn(v2.v[e], v3.v[e])));
                    }
#pragma unroll
                    for (int e = 0; e < RPL; ++e)
                        neg[e] += (int)(s0[e] == own_st[e]) + (int)(s1[e] == own_st[e]) + (int)(s2[e] == own_st[e]) + (int)(s3[e] == own_st[e]);
                    pk = nx;
                }
            } else if (PIGGY && count_now) {
                // scoring step: the sign bit of every gathered cosine is the neighbour's lattice state
#pragma unroll 1
                for (int gg = 0; gg < G; ++gg) {
                    const uint2 nx = next_group();
                    const PairPack<RPL> v0 = pairs_at(pk.x & 0xffffu), v1 = pairs_at(pk.x >> 16);
                    const PairPack<RPL> v2 = pairs_at(pk.y & 0xffffu), v3 = pairs_at(pk.y >> 16);
                    if (WEIGHTED) {
                        const float4 w4 = next_weights();
#pragma unroll
                        for (int e = 0; e < RPL; ++e) {
                            sum[e] = __ffma2_rn(make_float2(w4.x, w4.x), v0.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.y, w4.y), v1.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.z, w4.z), v2.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.w, w4.w), v3.v[e], sum[e]);
                            negw[e] += (__float_as_int(v0.v[e].x) < 0 ? w4.x : 0.f) + (__float_as_int(v1.v[e].x) < 0 ? w4.y : 0.f);
                            negw[e] += (__float_as_int(v2.v[e].x) < 0 ? w4.z : 0.f) + (__float_as_int(v3.v[e].x) < 0 ? w4.w : 0.f);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < RPL; ++e) {
                            sum[e] = __fadd2_rn(sum[e], __fadd2_rn(__fadd2_rn(v0.v[e], v1.v[e]), __fadd2_rn(v2.v[e], v3.v[e])));
                            neg[e] += (int)(__float_as_uint(v0.v[e].x) >> 31) + (int)(__float_as_uint(v1.v[e].x) >> 31);
                            neg[e] += (int)(__float_as_uint(v2.v[e].x) >> 31) + (int)(__float_as_uint(v3.v[e].x) >> 31);
                        }
                    }
                    pk = nx;
                }
            } else {
#pragma unroll 2
                for (int gg = 0; gg < G; ++gg) {
                    const uint2 nx = next_group();
                    const PairPack<RPL> v0 = pairs_at(pk.x & 0xffffu), v1 = pairs_at(pk.x >> 16);
                    const PairPack<RPL> v2 = pairs_at(pk.y & 0xffffu), v3 = pairs_at(pk.y >> 16);
                    if (WEIGHTED) {
                        const float4 w4 = next_weights();
#pragma unroll
                        for (int e = 0; e < RPL; ++e) {
                            sum[e] = __ffma2_rn(make_float2(w4.x, w4.x), v0.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.y, w4.y), v1.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.z, w4.z), v2.v[e], sum[e]);
                            sum[e] = __ffma2_rn(make_float2(w4.w, w4.w), v3.v[e], sum[e]);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < RPL; ++e)
                            sum[e] = __fadd2_rn(sum[e], __fadd2_rn(__fadd2_rn(v0.v[e], v1.v[e]), __fadd2_rn(v2.v[e], v3.v[e])));
                    }
                    pk = nx;
                }
            }
            if (draw && (warp & 1)) draw_noise();
            if (valid) {
                const PairPack<RPL> own = pairs_at(iRT);
                const uint32_t k = (iRT >> a.LRT) & 3u;
                int deg = 0;
                float wrow = 0.f;
                if (PIGGY && count_now && NMODE == 2) {
                    if (WEIGHTED) wrow = rowsum_lane[row * a.C];
                    else deg = (int)deg_lane[row * a.C];
                }
                float y[RPL];
#pragma unroll
                for (int e = 0; e < RPL; ++e) {
                    const float ci = own.v[e].x, si = own.v[e].y;
                    if (PIGGY && count_now && NMODE != 2) {
                        twice_cut[e] += neg[e];                          // equal-state neighbours: twice the conflicts
                    } else if (PIGGY && count_now) {   // differing neighbours: deg - neg if the row itself is in state 1
                        const bool own1 = __float_as_int(ci) < 0;        // the row's own state: the sign BIT
                        if (WEIGHTED) twice_cut_w[e] += own1 ? wrow - negw[e] : negw[e];
                        else twice_cut[e] += own1 ? deg - neg[e] : neg[e];
                    }
                    const float acc = si * sum[e].x - ci * sum[e].y;
                    float shil;
                    if (NMODE == 2) shil = si * ci;                              // hks holds 2 h ks
                    else shil = shil_term(p[e], si, ci, a.tc);
                    const float kick = (k & 2u) ? ((k & 1u) ? z[e][3] : z[e][2]) : ((k & 1u) ? z[e][1] : z[e][0]);
                    const float x = fmaf(a.hK, acc, fmaf(-hks, shil, fmaf(a.knsh, kick, p[e])));
                    float w = x - floorf(x);
                    y[e] = (w >= 1.0f) ? 0.0f : w;
                    if (!(fabsf(x) < INFINITY) && live[e])
                        flag_nonfinite(a.nonfinite, (uint64_t)step, (uint32_t)(rg0 + e), iRT >> a.LRT);
                }
                store_phi(iRT, y);
                if (STAGED) {
                    float s2[RPL], c2[RPL];
#pragma unroll
                    for (int e = 0; e < RPL; ++e) {
                        trig_turns_direct(y[e], s2[e], c2[e]);
                    }
                    if (RPL == 2) *reinterpret_cast<float4 *>(stage_g + iRT) = make_float4(c2[0], s2[0], c2[RPL - 1], s2[RPL - 1]);
                    else stage_g[iRT] = make_float2(c2[0], s2[0]);
                }
            }
        }
        if (count_now) {
            // `twice_cut` counted the state after step `pending_label`; cs still holds that state
            double tc[RPL];
#pragma unroll
            for (int e = 0; e < RPL; ++e) tc[e] = (WEIGHTED && NMODE == 2) ? (double)twice_cut_w[e] : (double)twice_cut[e];
            const double obj = 0.5 * tile_reduce_rpl<RPL>(tc, a.RT, a.LPS, part, tid, a.W);
            if (tid < a.RT) record_best(obj, pending_label);
            __syncthreads();
            publish_states();
            pending = false;
        }
        __syncthreads();

        // pass B: pairs (and state bytes) of the new phases -------------------------------------
        const bool score_after = is_sample || cadence_hit;
        if (STAGED) {
            // each lane copies back the pairs it staged itself (same thread wrote them: no fence needed)
#pragma unroll 4
            for (int row = 0; row < a.n_rows; ++row) {
                const uint32_t iRT = row_at(row);
                if (iRT < (uint32_t)a.nRT) {
                    if (RPL == 2) {
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(pair_addr<3>(iRT, cs32)), "l"(stage_g + iRT) : "memory");
                    } else {
                        float2 v;
                        asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(stage_g + iRT) : "memory");
                        sts_pair(pair_addr<3>(iRT, cs32), v.x, v.y);
                    }
                }
            }
            if (RPL == 2) asm volatile("cp.async.wait_all;" ::: "memory");
        } else {
#pragma unroll 1
            for (int row = 0; row < a.n_rows; ++row) {
                const uint32_t iRT = row_at(row);
                if (iRT < (uint32_t)a.nRT) {
                    float p[RPL];
                    load_phi(iRT, p);
                    float s[RPL], co[RPL];
#pragma unroll
                    for (int e = 0; e < RPL; ++e) {
                        trig_turns_direct(p[e], s[e], co[e]);
                    }
                    if (RPL == 2)
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(pair_addr<3>(iRT, cs32)), "f"(co[0]), "f"(s[0]),
                                     "f"(co[RPL - 1]), "f"(s[RPL - 1]) : "memory");
                    else
                        sts_pair(pair_addr<3>(iRT, cs32), co[0], s[0]);
                    if (score_after) {
#pragma unroll
                        for (int e = 0; e < RPL; ++e) sts_u8(st32 + iRT + e, state_of_phase(p[e]));
                    }
                }
            }
        }
        __syncthreads();

        if (is_sample) {
            score_current(step, a.sample_offset + sample_cur);
            ++sample_cur;
        } else if (cadence_hit) {
            if (PIGGY && a.piggy && step + 1 < a.step_end) {
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
        for (int i = tid; i < a.nRT; i += NT) slab[i] = phis[i];
    }
}

} // namespace oscb
