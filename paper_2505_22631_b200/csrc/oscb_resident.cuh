// oscb_resident.cuh -- the fused, persistent Euler-step kernel (K1 + K3 of SURVEY.md 2a).
//
// One CTA owns a tile of RT replicas for a whole run segment (thousands of Euler steps, one
// launch).  The (cos 2pi phi, sin 2pi phi) pairs of all n oscillators of those replicas stay
// in shared memory, laid out replica-minor
//     cs[j * RT + r]                (j = oscillator, r = replica inside the tile)
// so the RT lanes that share a neighbour read one contiguous RT*8-byte run.  A warp holds
// C = 32/RT "slots"; lane = slot_in_warp * RT + r.  A slot owns whole quads (four consecutive
// oscillators = one Philox block of normals) and walks them in `T` rounds.
//
// The neighbour lists are compiled on the host (oscb_resident_host.hpp) into a sliced-ELL
// stream: quads are sorted by degree and dealt to slots so that the C slots of a warp hold
// look-alike rows, the four rows of a quad are visited in descending-degree order, and for
// every (warp, round, row position) the C rows are padded to a common number G of 4-neighbour
// groups.  So the inner loop has a warp-uniform trip count, needs no row pointers, and reads
// the stream as one contiguous C*8-byte run per group:
//     stream[gp * C + slot_in_warp] = four u16 ids, each already multiplied by RT
// (ids >= n*RT name all-zero padding rows, one per shared-memory bank class, so padding never
// adds a bank conflict).  In the throughput mode the compiler also orders every row's
// neighbours so that the slots that share a shared-memory wavefront hit disjoint banks.
//
// Per step:
//   pass A: per own row, gather sum_j w (c_j, s_j) over the stream with packed f32x2 adds,
//           apply K, SHIL(ks(t)), Philox noise and the wrap, store the new phase (the tile's
//           phase slab [n][RT] in global memory, L2 resident -- one thread per element);
//   barrier (every gather of the old pairs is done)
//   pass B: recompute the (cos, sin) pairs of the own rows into shared memory; on scoring
//           steps also the lattice states (dynamics.py:203-213), one byte per cell;
//   barrier
//   scoring steps (reference cadence / trace samples): cut or conflict count over each own
//           row's neighbours j > i, fixed-order reduction per replica, strict-improvement best
//           tracking, optional energy sample (dynamics.py:370-384).
//
// Reference arithmetic restated: dynamics.py:166-172 (row update), :393-395 (trig), :83-88
// (schedule, float64 from the step index), :325-330/:404-410 (cadence and sample schedule;
// the sample step list is computed by the host with the reference's float arithmetic).
#pragma once
#include "oscb_device.cuh"

namespace oscb {

#define OSCB_PAD_ROWS 16 // all-zero rows after row n-1, one per bank class

struct ResidentArgs {
    int n;
    int R_real;                 // replicas that exist; tiles are padded up to RT
    int RT, log2RT;             // replicas per tile
    int C;                      // slots per warp = 32 / RT
    int T;                      // rounds (quads per slot)
    int W;                      // warps per CTA
    int n_group_rows;           // stream length in units of C groups (without the prefetch pad)
    const int *warp_start;      // [W]         first group row of each warp's stream
    const uint16_t *rows;       // [W*T*4*C]   own row * RT of (warp, round, position, slot); >= n*RT: none
    const uint32_t *ginfo;      // [W*T]       G of the four row positions, one byte each
    const uint2 *stream;        // [(n_group_rows + 1) * C]
    const void *wstream;        // [(n_group_rows + 1) * C * 4] weights in T (stream order); null = unit
    void *phi;                  // [tiles][n][RT] in T
    const uint64_t *seeds;      // [R_pad]
    long long step_begin, step_end;
    long long noise_step0;      // global step index of noise_host[0]
    double K, h, kn_sqrt_h, ks_max, ks_period;
    TrigConst tc;
    int noise_mode;
    const double *noise_host;   // [steps, R_real, n]
    long long cadence;          // <= 0: never score between samples
    const long long *sample_steps; // sorted global step indices; a sample is taken AFTER each
    int n_sample_steps;
    int sample_offset;          // trace column of sample_steps[0]
    int initial_sample;         // take the t = 0 sample (column 0) before step_begin
    int maximize;
    double *best_obj;           // [R_pad]
    uint8_t *best_states;       // [R_pad, n]
    double *energy;             // [R_pad, trace_stride]
    double *best_trace;         // [R_pad, trace_stride]
    long long trace_stride;
    long long *first_hit;       // [R_pad]
    int use_target;
    double target;
    unsigned long long *nonfinite;
};

// byte offsets of the regions inside dynamic shared memory (host and device agree on this)
struct ResidentSmem {
    size_t cs, st, rows, ginfo, part, misc, stream, wstream, total;
    __host__ __device__ static ResidentSmem make(int n, int RT, int C, int T, int W, size_t pair_bytes,
                                                 size_t weight_bytes, int n_group_rows, bool idx_smem, bool weighted)
    {
        ResidentSmem s;
        size_t o = 0;
        auto take = [&](size_t bytes) { size_t at = o; o += (bytes + 15) & ~(size_t)15; return at; };
        s.cs = take((size_t)(n + OSCB_PAD_ROWS) * RT * pair_bytes);
        s.st = take((size_t)(n + OSCB_PAD_ROWS) * RT);
        s.rows = take((size_t)W * T * 4 * C * 2);
        s.ginfo = take((size_t)W * T * 4);
        s.part = take((size_t)W * RT * 8);
        s.misc = take((size_t)RT * 16 + 32);
        s.stream = take(idx_smem ? (size_t)(n_group_rows + 1) * C * 8 : 0);
        s.wstream = take(idx_smem && weighted ? (size_t)(n_group_rows + 1) * C * 4 * weight_bytes : 0);
        s.total = o;
        return s;
    }
};

// Sum `v` over all threads of the CTA that share replica r = lane & (RT-1), in a fixed order
// (deterministic).  Result valid in threads tid < RT.  Two barriers inside.
__device__ __forceinline__ double tile_reduce(double v, int RT, double *part, int tid, int nwarps)
{
    const int lane = tid & 31, warp = tid >> 5;
    for (int off = 16; off >= RT; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane < RT) part[warp * RT + lane] = v;
    __syncthreads();
    double tot = 0.0;
    if (tid < RT)
        for (int w = 0; w < nwarps; ++w) tot += part[w * RT + tid];
    __syncthreads();
    return tot;
}

// shared-memory pair load at a 32-bit shared address; the address of row id*RT is one IMAD/LEA
// off the lane's base (PTX mad.lo keeps ptxas from splitting it into shift + mask + add)
__device__ __forceinline__ void lds_pair(uint32_t addr, float2 &v)
{
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
}
__device__ __forceinline__ void lds_pair(uint32_t addr, double2 &v)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
}
template <int PSH> __device__ __forceinline__ uint32_t pair_addr(uint32_t id, uint32_t base)
{
    uint32_t a;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(id), "n"(1 << PSH), "r"(base));
    return a;
}

// packed pair arithmetic: one FADD2 / FFMA2 per (cos, sin) pair on sm_100a
__device__ __forceinline__ float2 pair_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ double2 pair_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 pair_fma(float w, float2 v, float2 acc) { return __ffma2_rn(make_float2(w, w), v, acc); }
__device__ __forceinline__ double2 pair_fma(double w, double2 v, double2 acc)
{
    return make_double2(fma(w, v.x, acc.x), fma(w, v.y, acc.y));
}

template <typename T, int MAXT, bool IDX_SMEM, bool WEIGHTED, bool STRICT>
__global__ void __launch_bounds__(MAXT, 1) k_resident(const ResidentArgs a)
{
    using T2 = typename Vec2<T>::type;
    constexpr int PSH = sizeof(T2) == 8 ? 3 : 4;   // log2 bytes per pair
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, NT = blockDim.x, W = a.W;
    const int RT = a.RT, n = a.n, C = a.C, TR = a.T;
    const ResidentSmem L = ResidentSmem::make(n, RT, C, TR, W, sizeof(T2), sizeof(T), a.n_group_rows, IDX_SMEM, WEIGHTED);
    T2 *cs = reinterpret_cast<T2 *>(smem_raw + L.cs);
    uint8_t *stb = smem_raw + L.st;
    uint16_t *rows_s = reinterpret_cast<uint16_t *>(smem_raw + L.rows);
    uint32_t *ginfo_s = reinterpret_cast<uint32_t *>(smem_raw + L.ginfo);
    double *part = reinterpret_cast<double *>(smem_raw + L.part);
    double *best_s = reinterpret_cast<double *>(smem_raw + L.misc);          // [RT]
    int *improved_s = reinterpret_cast<int *>(smem_raw + L.misc + RT * 8);   // [RT]
    double *ks_s = reinterpret_cast<double *>(smem_raw + L.misc + RT * 16);  // [2]
    const uint2 *stream = IDX_SMEM ? reinterpret_cast<const uint2 *>(smem_raw + L.stream) : a.stream;
    const T *wstream = (IDX_SMEM && WEIGHTED) ? reinterpret_cast<const T *>(smem_raw + L.wstream)
                                              : reinterpret_cast<const T *>(a.wstream);

    const int lane = tid & 31, warp = tid >> 5;
    const int r = lane & (RT - 1), c = lane >> a.log2RT;
    const int tile = blockIdx.x;
    const int rg = tile * RT + r;                  // global replica index
    const bool live = rg < a.R_real;
    const uint64_t seed = a.seeds[rg];
    T *phi = reinterpret_cast<T *>(a.phi) + (size_t)tile * n * RT + r;       // + (row * RT)
    unsigned char *cs_lane = smem_raw + L.cs + r * sizeof(T2);               // + (row * RT) << PSH
    const uint32_t cs_lane32 = (uint32_t)__cvta_generic_to_shared(cs_lane);  // same, as a shared address
    auto pair_at = [&](uint32_t idRT) -> T2 { T2 v; lds_pair(pair_addr<PSH>(idRT, cs_lane32), v); return v; };
    uint8_t *st_lane = stb + r;                                              // + (row * RT)
    const int nRT = n * RT;

    // ---- prologue: stage the plan, build (cos, sin) of the current phases --------------------
    for (int q = tid; q < W * TR * 4 * C; q += NT) rows_s[q] = a.rows[q];
    for (int q = tid; q < W * TR; q += NT) ginfo_s[q] = a.ginfo[q];
    if (IDX_SMEM) {
        uint2 *dst = reinterpret_cast<uint2 *>(smem_raw + L.stream);
        for (int q = tid; q < (a.n_group_rows + 1) * C; q += NT) dst[q] = a.stream[q];
        if (WEIGHTED) {
            T *wd = reinterpret_cast<T *>(smem_raw + L.wstream);
            const T *ws = reinterpret_cast<const T *>(a.wstream);
            for (int q = tid; q < (a.n_group_rows + 1) * C * 4; q += NT) wd[q] = ws[q];
        }
    }
    {
        const T *slab = reinterpret_cast<const T *>(a.phi) + (size_t)tile * n * RT;
        for (int q = tid; q < nRT; q += NT) {
            T s, co;
            phase_trig(slab[q], s, co);
            T2 v; v.x = co; v.y = s;
            cs[q] = v;
        }
        for (int q = tid; q < OSCB_PAD_ROWS * RT; q += NT) {      // padding rows: zero pairs, state 255
            T2 zero; zero.x = T(0); zero.y = T(0);
            cs[nRT + q] = zero;
            stb[nRT + q] = 255;
        }
    }
    if (tid < RT) {
        best_s[tid] = a.best_obj[tile * RT + tid];
        improved_s[tid] = 0;
    }
    if (tid == 0) ks_s[a.step_begin & 1] = ks_value(a.ks_max, a.ks_period, (double)a.step_begin * a.h);
    const int gp0 = a.warp_start[warp];
    __syncthreads();

    // own row (pre-multiplied by RT) of (round t, position kk); >= nRT when the slot has none
    auto own_row = [&](int t, int kk) -> int { return rows_s[((warp * TR + t) * 4 + kk) * C + c]; };

    // lattice states of the own rows -> stb
    auto write_states = [&]() {
        for (int t = 0; t < TR; ++t)
            for (int kk = 0; kk < 4; ++kk) {
                const int iRT = own_row(t, kk);
                if (iRT < nRT) st_lane[iRT] = (uint8_t)threshold_state((double)phi[iRT], a.tc.n_states);
            }
    };

    // score the state currently in cs / stb; sample_col >= 0 also records that trace column
    auto score_current = [&](long long step_label, int sample_col) {
        double obj_part = 0.0, en_part = 0.0;
        int gp = gp0;
        for (int t = 0; t < TR; ++t) {
            const uint32_t g4 = ginfo_s[warp * TR + t];
            for (int kk = 0; kk < 4; ++kk) {
                const int G = (g4 >> (8 * kk)) & 0xFF;
                const int iRT = own_row(t, kk);
                if (iRT < nRT) {
                    const uint32_t si = st_lane[iRT];
                    const T2 own = pair_at(iRT);
                    int count = 0;
                    double wsum = 0.0;
                    for (int g = 0; g < G; ++g) {
                        const uint2 pk = stream[(gp + g) * C + c];
                        const int jj[4] = {(int)(pk.x & 0xffffu), (int)(pk.x >> 16), (int)(pk.y & 0xffffu), (int)(pk.y >> 16)};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int jRT = jj[u];
                            if (jRT > iRT && jRT < nRT) {                  // canonical pairs i < j only
                                const bool same = st_lane[jRT] == si;
                                const bool hit = a.maximize ? !same : same;
                                if (WEIGHTED) {
                                    const double w = (double)wstream[((size_t)(gp + g) * C + c) * 4 + u];
                                    if (hit) wsum += a.maximize ? w : 1.0;
                                    if (sample_col >= 0) {
                                        const T2 v = pair_at(jRT);
                                        en_part += w * ((double)own.x * (double)v.x + (double)own.y * (double)v.y);
                                    }
                                } else {
                                    count += hit ? 1 : 0;
                                    if (sample_col >= 0) {
                                        const T2 v = pair_at(jRT);
                                        en_part += (double)own.x * (double)v.x + (double)own.y * (double)v.y;
                                    }
                                }
                            }
                        }
                    }
                    obj_part += WEIGHTED ? wsum : (double)count;
                }
                gp += G;
            }
        }
        const double obj = tile_reduce(obj_part, RT, part, tid, W);
        if (tid < RT) {
            const double b = best_s[tid];
            const bool better = a.maximize ? (obj > b) : (obj < b);
            improved_s[tid] = better ? 1 : 0;
            if (better) {
                best_s[tid] = obj;
                const int gi = tile * RT + tid;
                if (a.use_target && a.first_hit[gi] < 0 && (a.maximize ? (obj >= a.target) : (obj <= a.target)))
                    a.first_hit[gi] = step_label;
            }
        }
        __syncthreads();
        if (improved_s[r] && live) {           // strict improvement: publish this replica's states
            uint8_t *dst = a.best_states + (size_t)rg * n;
            for (int t = 0; t < TR; ++t)
                for (int kk = 0; kk < 4; ++kk) {
                    const int iRT = own_row(t, kk);
                    if (iRT < nRT) dst[iRT >> a.log2RT] = st_lane[iRT];
                }
        }
        if (sample_col >= 0) {
            const double en = tile_reduce(en_part, RT, part, tid, W);
            if (tid < RT) {
                const size_t gi = (size_t)(tile * RT + tid);
                a.energy[gi * a.trace_stride + sample_col] = en;
                a.best_trace[gi * a.trace_stride + sample_col] = best_s[tid];
            }
        }
        __syncthreads();
    };

    int sample_cur = 0; // cursor into sample_steps
    while (sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] < a.step_begin) ++sample_cur;

    if (a.initial_sample) {
        write_states();
        __syncthreads();
        score_current(-1, 0);
    }

    const T hK = (T)(a.h * a.K), knsh = (T)a.kn_sqrt_h;

    // ---- time loop ---------------------------------------------------------------------------
#pragma unroll 1
    for (long long step = a.step_begin; step < a.step_end; ++step) {
        const double ks = ks_s[step & 1];
        const T hks = (T)(a.h * ks);
        const bool is_sample = sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] == step;
        const bool do_score = is_sample || (a.cadence > 0 && step % a.cadence == 0);
        // pass A: gather + update.  The stream of a warp is contiguous, so the next group is
        // always prefetched one iteration ahead (the pad row covers the last one).
        const uint2 *sp = stream + (size_t)gp0 * C + c;
        const T *wp = WEIGHTED ? wstream + ((size_t)gp0 * C + c) * 4 : nullptr;
        uint2 pk = *sp;
#pragma unroll 1
        for (int t = 0; t < TR; ++t) {
            const uint32_t g4 = ginfo_s[warp * TR + t];
            T z[4] = {T(0), T(0), T(0), T(0)};
            if (a.noise_mode == 0) {
                const int first = own_row(t, 0);
                if (first < nRT) normals4(noise_block(seed, (uint64_t)step, (uint32_t)(first >> a.log2RT) >> 2), z);
            }
#pragma unroll 1
            for (int kk = 0; kk < 4; ++kk) {
                const int G = (g4 >> (8 * kk)) & 0xFF;      // warp-uniform trip count
                const int iRT = own_row(t, kk);
                const bool valid = iRT < nRT;
                const T p = valid ? phi[iRT] : T(0);
                const T2 own = pair_at(iRT);
                const T ci = own.x, si = own.y;
                T acc;
                if (STRICT) {
                    // reference order: acc += w * (s_i c_j - c_i s_j), one neighbour at a time
                    double accd = 0.0;
                    for (int g = 0; g < G; ++g) {
                        sp += C;
                        const uint2 nx = *sp;
                        const uint32_t jj[4] = {pk.x & 0xffffu, pk.x >> 16, pk.y & 0xffffu, pk.y >> 16};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const T2 v = pair_at(jj[u]);
                            const double w = WEIGHTED ? (double)wp[u] : 1.0;
                            const double term = __dsub_rn(__dmul_rn((double)si, (double)v.x), __dmul_rn((double)ci, (double)v.y));
                            accd = __dadd_rn(accd, __dmul_rn(w, term));
                        }
                        if (WEIGHTED) wp += 4 * C;
                        pk = nx;
                    }
                    acc = (T)accd;
                } else {
                    T2 sum; sum.x = T(0); sum.y = T(0);
#pragma unroll 2
                    for (int g = 0; g < G; ++g) {
                        sp += C;
                        const uint2 nx = *sp;
                        const T2 v0 = pair_at(pk.x & 0xffffu), v1 = pair_at(pk.x >> 16);
                        const T2 v2 = pair_at(pk.y & 0xffffu), v3 = pair_at(pk.y >> 16);
                        if (WEIGHTED) {
                            sum = pair_fma(wp[0], v0, sum);
                            sum = pair_fma(wp[1], v1, sum);
                            sum = pair_fma(wp[2], v2, sum);
                            sum = pair_fma(wp[3], v3, sum);
                            wp += 4 * C;
                        } else {
                            sum = pair_add(sum, pair_add(pair_add(v0, v1), pair_add(v2, v3)));
                        }
                        pk = nx;
                    }
                    acc = si * sum.x - ci * sum.y;
                }
                if (valid) {
                    const int i = iRT >> a.log2RT, k = i & 3;
                    const T shil = shil_term(p, si, ci, a.tc);
                    T kick = (k == 0) ? z[0] : (k == 1) ? z[1] : (k == 2) ? z[2] : z[3];
                    if (a.noise_mode == 1)
                        kick = live ? (T)a.noise_host[((size_t)(step - a.noise_step0) * a.R_real + rg) * n + i] : T(0);
                    T x;
                    if (STRICT) {
                        const double drift = __dsub_rn(__dmul_rn(a.K, (double)acc), __dmul_rn(ks, (double)shil));
                        x = (T)__dadd_rn(__dadd_rn((double)p, __dmul_rn(a.h, drift)), __dmul_rn(a.kn_sqrt_h, (double)kick));
                    } else {
                        x = fma(hK, acc, fma(-hks, shil, fma(knsh, kick, p)));
                    }
                    if (!isfinite(x) && live) flag_nonfinite(a.nonfinite, (uint64_t)step, (uint32_t)rg, (uint32_t)i);
                    phi[iRT] = wrap_unit(x);
                }
            }
        }
        if (tid == 0) ks_s[(step + 1) & 1] = ks_value(a.ks_max, a.ks_period, (double)(step + 1) * a.h);
        __syncthreads();
        // pass B: (cos, sin) of the new phases; lattice states when this step is scored
#pragma unroll 1
        for (int t = 0; t < TR; ++t) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int iRT = own_row(t, kk);
                if (iRT < nRT) {
                    const T p = phi[iRT];
                    T s, co;
                    phase_trig(p, s, co);
                    T2 v; v.x = co; v.y = s;
                    *reinterpret_cast<T2 *>(cs_lane + ((size_t)iRT << PSH)) = v;
                    if (do_score) st_lane[iRT] = (uint8_t)threshold_state((double)p, a.tc.n_states);
                }
            }
        }
        __syncthreads();
        // scoring schedule (dynamics.py:404-410)
        if (is_sample) {
            score_current(step, a.sample_offset + sample_cur);
            ++sample_cur;
        } else if (do_score) {
            score_current(step, -1);
        }
    }
    if (tid < RT) a.best_obj[tile * RT + tid] = best_s[tid];
}

// host layout [R, n] float64  <->  tile slabs [tiles][n][RT] in T (dead replicas read as 0)
template <typename T>
__global__ void k_to_tile_layout(const double *__restrict__ src, T *__restrict__ dst, int n, int R, int RT, long long total)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= total) return;
    const int r = (int)(q % RT);
    const long long rest = q / RT;
    const int i = (int)(rest % n), tile = (int)(rest / n);
    const int rg = tile * RT + r;
    dst[q] = rg < R ? (T)src[(long long)rg * n + i] : T(0);
}
template <typename T>
__global__ void k_from_tile_layout(const T *__restrict__ src, double *__restrict__ dst, int n, int R, int RT)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n * R) return;
    const int rg = (int)(q / n), i = (int)(q - (long long)rg * n);
    const int tile = rg / RT, r = rg - tile * RT;
    dst[q] = (double)src[((long long)tile * n + i) * RT + r];
}

} // namespace oscb
