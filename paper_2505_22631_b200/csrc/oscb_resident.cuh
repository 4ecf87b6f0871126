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
//     stream[gp * C + slot_in_warp] = four u16 neighbour ids   (dummy id n -> a zero pair)
//
// Per step:
//   pass A: per own row, gather sum_j w c_j / sum_j w s_j over the stream, apply
//           K, SHIL(ks(t)), Philox noise and the wrap, store the new phase (the tile's phase
//           slab [n][RT] in global memory, L2 resident -- each element is touched by one thread);
//   barrier (every gather of the old pairs is done)
//   pass B: recompute the (cos, sin) pairs of the own rows into shared memory; on scoring
//           steps also the lattice states (dynamics.py:203-213), bit-packed;
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

struct ResidentArgs {
    int n;
    int R_real;                 // replicas that exist; tiles are padded up to RT
    int RT, log2RT;             // replicas per tile
    int C;                      // slots per warp = 32 / RT
    int T;                      // rounds (quads per slot)
    int W;                      // warps per CTA
    int SB, wpr;                // state bits per cell, 32-bit state words per row
    int n_group_rows;           // stream length in units of C groups
    const int *warp_start;      // [W]      first group row of each warp's stream
    const int *quad_of;         // [W*T*C]  quad | visiting order << 24, or -1
    const uint32_t *ginfo;      // [W*T]    G of the four row positions, one byte each
    const uint2 *stream;        // [n_group_rows * C]
    const void *wstream;        // [n_group_rows * C * 4] weights in T (stream order); null = unit
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
    size_t cs, st, quad, ginfo, wstart, part, misc, stream, wstream, total;
    __host__ __device__ static ResidentSmem make(int n, int RT, int C, int T, int W, int wpr, size_t pair_bytes,
                                                 size_t weight_bytes, int n_group_rows, bool idx_smem, bool weighted)
    {
        ResidentSmem s;
        size_t o = 0;
        auto take = [&](size_t bytes) { size_t at = o; o += (bytes + 15) & ~(size_t)15; return at; };
        s.cs = take((size_t)(n + 1) * RT * pair_bytes);
        s.st = take((size_t)(n + 1) * wpr * 4);
        s.quad = take((size_t)W * T * C * 4);
        s.ginfo = take((size_t)W * T * 4);
        s.wstart = take((size_t)W * 4);
        s.part = take((size_t)W * RT * 8);
        s.misc = take((size_t)RT * 16 + 32);
        s.stream = take(idx_smem ? (size_t)n_group_rows * C * 8 : 0);
        s.wstream = take(idx_smem && weighted ? (size_t)n_group_rows * C * 4 * weight_bytes : 0);
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

template <typename T, int MAXT, bool IDX_SMEM, bool WEIGHTED, bool STRICT>
__global__ void __launch_bounds__(MAXT, 1) k_resident(const ResidentArgs a)
{
    using T2 = typename Vec2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, NT = blockDim.x, W = a.W;
    const int RT = a.RT, n = a.n, C = a.C, TR = a.T, SB = a.SB, wpr = a.wpr;
    const ResidentSmem L = ResidentSmem::make(n, RT, C, TR, W, wpr, sizeof(T2), sizeof(T), a.n_group_rows, IDX_SMEM, WEIGHTED);
    T2 *cs = reinterpret_cast<T2 *>(smem_raw + L.cs);
    uint32_t *stw = reinterpret_cast<uint32_t *>(smem_raw + L.st);
    int *quad_s = reinterpret_cast<int *>(smem_raw + L.quad);
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
    T *phi = reinterpret_cast<T *>(a.phi) + (size_t)tile * n * RT;
    const uint32_t smask = (SB >= 32) ? 0xffffffffu : ((1u << SB) - 1u);
    const int sshift = (r * SB) & 31, sword = (r * SB) >> 5;
    int cells_per_word = 32 / SB;                  // lanes whose cells share one state word
    if (cells_per_word > RT) cells_per_word = RT;

    // ---- prologue: stage the plan, build (cos, sin) of the current phases --------------------
    for (int q = tid; q < W * TR * C; q += NT) quad_s[q] = a.quad_of[q];
    for (int q = tid; q < W * TR; q += NT) ginfo_s[q] = a.ginfo[q];
    if (IDX_SMEM) {
        uint2 *dst = reinterpret_cast<uint2 *>(smem_raw + L.stream);
        for (int q = tid; q < a.n_group_rows * C; q += NT) dst[q] = a.stream[q];
        if (WEIGHTED) {
            T *wd = reinterpret_cast<T *>(smem_raw + L.wstream);
            const T *ws = reinterpret_cast<const T *>(a.wstream);
            for (int q = tid; q < a.n_group_rows * C * 4; q += NT) wd[q] = ws[q];
        }
    }
    for (int q = tid; q < n * RT; q += NT) {
        T s, co;
        phase_trig(phi[q], s, co);
        T2 v; v.x = co; v.y = s;
        cs[q] = v;
    }
    if (tid < RT) {
        T2 zero; zero.x = T(0); zero.y = T(0);
        cs[n * RT + tid] = zero;                   // the dummy neighbour used by stream padding
        best_s[tid] = a.best_obj[tile * RT + tid];
        improved_s[tid] = 0;
    }
    if (tid == 0) ks_s[a.step_begin & 1] = ks_value(a.ks_max, a.ks_period, (double)a.step_begin * a.h);
    const int gp0 = a.warp_start[warp];
    __syncthreads();

    // own-row iteration helpers -------------------------------------------------------------
    // quad word of (round t): quad index | order << 20, or -1 when the slot has no quad
    auto quad_word = [&](int t) -> int { return quad_s[(warp * TR + t) * C + c]; };

    // lattice states of the own rows -> stw (bit-packed, one word group per row)
    auto write_states = [&]() {
        for (int t = 0; t < TR; ++t) {
            const int qw = quad_word(t);
            const int quad = qw & 0xFFFFF;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * quad + k;
                const bool valid = qw >= 0 && i < n;
                uint32_t v = 0;
                if (valid) v = (uint32_t)threshold_state((double)phi[i * RT + r], a.tc.n_states) << sshift;
                for (int off = 1; off < cells_per_word; off <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, off);
                if (valid && (r & (cells_per_word - 1)) == 0) stw[i * wpr + sword] = v;
            }
        }
    };
    auto load_state = [&](int j) -> uint32_t { return (stw[j * wpr + sword] >> sshift) & smask; };

    // score the state currently in cs / phi / stw; sample_col >= 0 also records that trace column
    auto score_current = [&](long long step_label, int sample_col) {
        double obj_part = 0.0, en_part = 0.0;
        int gp = gp0;
        for (int t = 0; t < TR; ++t) {
            const int qw = quad_word(t);
            const uint32_t g4 = ginfo_s[warp * TR + t];
            const int quad = qw & 0xFFFFF, order = (qw >> 20) & 0xFF;
            for (int kk = 0; kk < 4; ++kk) {
                const int G = (g4 >> (8 * kk)) & 0xFF;
                const int i = 4 * quad + ((order >> (2 * kk)) & 3);
                const bool valid = qw >= 0 && i < n;
                if (valid) {
                    const uint32_t si = load_state(i);
                    const T2 own = cs[i * RT + r];
                    for (int g = 0; g < G; ++g) {
                        const uint2 pk = stream[(gp + g) * C + c];
                        const int jj[4] = {(int)(pk.x & 0xffffu), (int)(pk.x >> 16), (int)(pk.y & 0xffffu), (int)(pk.y >> 16)};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int j = jj[u];
                            if (j > i && j < n) {
                                const double w = WEIGHTED ? (double)wstream[((size_t)(gp + g) * C + c) * 4 + u] : 1.0;
                                const bool same = load_state(j) == si;
                                if (a.maximize) { if (!same) obj_part += w; }
                                else            { if (same) obj_part += 1.0; }
                                if (sample_col >= 0) {
                                    const T2 v = cs[j * RT + r];
                                    en_part += w * ((double)own.x * (double)v.x + (double)own.y * (double)v.y);
                                }
                            }
                        }
                    }
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
            for (int t = 0; t < TR; ++t) {
                const int qw = quad_word(t);
                if (qw < 0) continue;
                const int quad = qw & 0xFFFFF;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = 4 * quad + k;
                    if (i < n) dst[i] = (uint8_t)load_state(i);
                }
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
        const bool do_score = is_sample || (a.cadence > 0 && (step - a.step_begin + a.step_begin) % a.cadence == 0);
        int gp = gp0;
        // pass A: gather + update
#pragma unroll 1
        for (int t = 0; t < TR; ++t) {
            const int qw = quad_word(t);
            const uint32_t g4 = ginfo_s[warp * TR + t];
            const int quad = qw & 0xFFFFF, order = (qw >> 20) & 0xFF;
            T z[4] = {T(0), T(0), T(0), T(0)};
            if (a.noise_mode == 0 && qw >= 0) normals4(noise_block(seed, (uint64_t)step, (uint32_t)quad), z);
#pragma unroll 1
            for (int kk = 0; kk < 4; ++kk) {
                const int G = (g4 >> (8 * kk)) & 0xFF;      // warp-uniform trip count
                const int k = (order >> (2 * kk)) & 3;
                const int i = 4 * quad + k;
                const bool valid = qw >= 0 && i < n;
                const int io = valid ? i : n;               // invalid rows read the zero pair
                const T p = valid ? phi[i * RT + r] : T(0);
                const T2 own = cs[io * RT + r];
                const T ci = own.x, si = own.y;
                T acc;
                if (STRICT) {
                    // reference order: acc += w * (s_i c_j - c_i s_j), one neighbour at a time
                    double accd = 0.0;
                    for (int g = 0; g < G; ++g) {
                        const uint2 pk = stream[(gp + g) * C + c];
                        const int jj[4] = {(int)(pk.x & 0xffffu), (int)(pk.x >> 16), (int)(pk.y & 0xffffu), (int)(pk.y >> 16)};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const T2 v = cs[jj[u] * RT + r];
                            const double w = WEIGHTED ? (double)wstream[((size_t)(gp + g) * C + c) * 4 + u] : 1.0;
                            const double term = __dsub_rn(__dmul_rn((double)si, (double)v.x), __dmul_rn((double)ci, (double)v.y));
                            accd = __dadd_rn(accd, __dmul_rn(w, term));
                        }
                    }
                    acc = (T)accd;
                } else {
                    T ac = T(0), as = T(0);
                    for (int g = 0; g < G; ++g) {
                        const uint2 pk = stream[(gp + g) * C + c];
                        const T2 v0 = cs[(int)(pk.x & 0xffffu) * RT + r];
                        const T2 v1 = cs[(int)(pk.x >> 16) * RT + r];
                        const T2 v2 = cs[(int)(pk.y & 0xffffu) * RT + r];
                        const T2 v3 = cs[(int)(pk.y >> 16) * RT + r];
                        if (WEIGHTED) {
                            const T *wp = wstream + ((size_t)(gp + g) * C + c) * 4;
                            const T w0 = wp[0], w1 = wp[1], w2 = wp[2], w3 = wp[3];
                            ac = fma(w0, v0.x, ac); as = fma(w0, v0.y, as);
                            ac = fma(w1, v1.x, ac); as = fma(w1, v1.y, as);
                            ac = fma(w2, v2.x, ac); as = fma(w2, v2.y, as);
                            ac = fma(w3, v3.x, ac); as = fma(w3, v3.y, as);
                        } else {
                            ac += (v0.x + v1.x) + (v2.x + v3.x);
                            as += (v0.y + v1.y) + (v2.y + v3.y);
                        }
                    }
                    acc = si * ac - ci * as;
                }
                gp += G;
                if (valid) {
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
                    phi[i * RT + r] = wrap_unit(x);
                }
            }
        }
        if (tid == 0) ks_s[(step + 1) & 1] = ks_value(a.ks_max, a.ks_period, (double)(step + 1) * a.h);
        __syncthreads();
        // pass B: (cos, sin) of the new phases; lattice states when this step is scored
#pragma unroll 1
        for (int t = 0; t < TR; ++t) {
            const int qw = quad_word(t);
            const int quad = qw & 0xFFFFF;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * quad + k;
                const bool valid = qw >= 0 && i < n;
                T p = T(0);
                if (valid) {
                    p = phi[i * RT + r];
                    T s, co;
                    phase_trig(p, s, co);
                    T2 v; v.x = co; v.y = s;
                    cs[i * RT + r] = v;
                }
                if (do_score) {                            // CTA-uniform branch
                    uint32_t v = 0;
                    if (valid) v = (uint32_t)threshold_state((double)p, a.tc.n_states) << sshift;
                    for (int off = 1; off < cells_per_word; off <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, off);
                    if (valid && (r & (cells_per_word - 1)) == 0) stw[i * wpr + sword] = v;
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
