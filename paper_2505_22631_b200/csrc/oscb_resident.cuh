// oscb_resident.cuh -- the fused, persistent Euler-step kernel (K1 + K3 of SURVEY.md 2a).
//
// One CTA owns a tile of RT replicas for the WHOLE run segment.  The (cos 2pi phi, sin 2pi phi)
// pairs of all n oscillators of those replicas stay in shared memory, laid out
//     cs[j * RT + r]                (j = oscillator, r = replica inside the tile)
// so a warp's neighbour gather reads RT consecutive pairs per neighbour.  Thread t owns replica
// r = t % RT and the rows of the quads  slot, slot + nslots, ...  (slot = t / RT, a quad = four
// consecutive oscillators = one Philox block of normals).  The neighbour lists are stored as a
// per-slot STREAM in exactly the order the owning threads walk them: groups of four u16 ids
// (dummy id n pads a row to a multiple of four and points at a zero (cos, sin) pair), bit 15 of
// the first id marks a row's last group, so the inner loop needs no row pointers at all.
//
// Per step:
//     pass A: walk the stream, accumulate sum w c_j / sum w s_j, apply SHIL + schedule +
//             Philox noise + wrap, store the new phase (own element of the tile's L2-resident
//             phase slab);
//     barrier (all gathers of the old pairs are done)
//     pass B: recompute (cos, sin) of the new phases into shared memory;
//     barrier
//     scoring steps only (reference cadence): round to lattice states (dynamics.py:203-213,
//             bit-packed in shared memory), cut / conflict count over each row's j > i
//             neighbours, fixed-order reduction per replica, strict-improvement best tracking,
//             optional energy sample (dynamics.py:370-384).
// HBM traffic per step is the phase slab read+write (8 B per oscillator-replica in fp32),
// which stays in the 126 MB L2; the graph stream is read once per launch when it fits in
// shared memory next to the pairs, else once per step through L2.
//
// Reference arithmetic restated: dynamics.py:166-172 (row update), :393-395 (trig), :83-88
// (schedule, evaluated in fp64 from the step index), :325-330/:404-410 (scoring cadence and
// sample scheduling -- the sample step list is computed by the host with the reference's exact
// float arithmetic and passed in).
#pragma once
#include "oscb_device.cuh"

namespace oscb {

struct ResidentArgs {
    int n;
    int R_real;                 // replicas that exist; tiles are padded up to RT
    int RT, log2RT;
    int state_bits;             // 1, 2, 4 or 8 bits per lattice state in shared memory
    int n_groups;               // total 4-entry groups in the stream
    const int *slot_start;      // [nslots] first group of each slot's stream
    const uint2 *idx4;          // [n_groups] four u16 neighbour ids; bit 15 of id 0 = row end
    const void *wstream;        // [4*n_groups] weights in T (stream order), null for unit weights
    void *phi;                  // [tiles][n][RT] in T
    const uint64_t *seeds;      // [R_pad]
    long long step_begin, step_end;
    long long noise_step0;      // global step index of noise_host[0]
    double K, h, kn_sqrt_h, ks_max, ks_period;
    TrigConst tc;
    int noise_mode;
    const double *noise_host;   // [steps, R_real, n]
    long long cadence;          // <= 0: never score between samples
    const long long *sample_steps; // sorted; a sample is taken AFTER these steps
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

template <typename T> struct ResidentSmem {
    using T2 = typename Vec2<T>::type;
    size_t cs, idx, st, part, misc, total; // byte offsets inside dynamic shared memory
    __host__ __device__ static ResidentSmem make(int n, int RT, int n_groups, bool idx_smem,
                                                 int nthreads, int state_bits)
    {
        ResidentSmem s;
        const int quads = (n + 3) >> 2, nslots = nthreads / RT;
        const int iters = (quads + nslots - 1) / nslots;
        size_t o = 0;
        s.cs = o;   o += (size_t)(n + 1) * RT * sizeof(T2);
        s.idx = o;  o += idx_smem ? (size_t)n_groups * sizeof(uint2) : 0;
        s.st = o;   o += (((size_t)iters * 4 * nthreads * state_bits / 8) + 15) & ~(size_t)15;
        s.part = o; o += (size_t)(nthreads / 32) * RT * sizeof(double);
        s.misc = o; o += (size_t)RT * 16 + 64;
        s.total = o;
        return s;
    }
};

// reduce `v` over all threads of the CTA that share replica r = tid & (RT-1), in a fixed order
// (deterministic); result valid in threads tid < RT.  Two barriers inside.
__device__ __forceinline__ double tile_reduce(double v, int RT, double *part, int tid, int nwarps)
{
    const int lane = tid & 31, warp = tid >> 5;
    for (int off = 16; off >= RT; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane < RT) part[warp * RT + lane] = v; // RT <= 32; lane == r for these lanes
    __syncthreads();
    double tot = 0.0;
    if (tid < RT)
        for (int w = 0; w < nwarps; ++w) tot += part[w * RT + tid];
    __syncthreads();
    return tot;
}

template <typename T, bool IDX_SMEM, bool WEIGHTED, bool STRICT>
__global__ void __launch_bounds__(1024, 1) k_resident(ResidentArgs a)
{
    using T2 = typename Vec2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, NT = blockDim.x, nwarps = NT >> 5;
    const int RT = a.RT, n = a.n, SB = a.state_bits;
    const ResidentSmem<T> L = ResidentSmem<T>::make(n, RT, a.n_groups, IDX_SMEM, NT, SB);
    T2 *cs = reinterpret_cast<T2 *>(smem_raw + L.cs);
    uint32_t *stw = reinterpret_cast<uint32_t *>(smem_raw + L.st);
    double *part = reinterpret_cast<double *>(smem_raw + L.part);
    double *best_s = reinterpret_cast<double *>(smem_raw + L.misc);           // [RT]
    int *improved_s = reinterpret_cast<int *>(smem_raw + L.misc + RT * 8);    // [RT]
    double *ks_s = reinterpret_cast<double *>(smem_raw + L.misc + RT * 16);   // [2]
    const uint2 *idx4 = IDX_SMEM ? reinterpret_cast<const uint2 *>(smem_raw + L.idx) : a.idx4;
    const T *wstream = reinterpret_cast<const T *>(a.wstream);

    const int r = tid & (RT - 1), slot = tid >> a.log2RT, nslots = NT >> a.log2RT;
    const int log2ns = 31 - __clz(nslots), log2NT = 31 - __clz(NT);
    const int tile = blockIdx.x;
    const int rg = tile * RT + r;                 // global replica index
    const bool live = rg < a.R_real;
    const uint64_t seed = a.seeds[rg];
    T *phi = reinterpret_cast<T *>(a.phi) + (size_t)tile * n * RT;
    const int quads = (n + 3) >> 2;
    const int g_start = a.slot_start[slot];
    const uint32_t smask = (SB == 8) ? 0xffu : ((1u << SB) - 1u);
    const int lanes_per_word = 32 / SB;

    // state cell of (row j, replica rr): rows are numbered in the order their owners visit them
    auto state_cell = [&](int j, int rr) -> int {
        const int qd = j >> 2;
        return ((((qd >> log2ns) << 2) + (j & 3)) << log2NT) + ((qd & (nslots - 1)) << a.log2RT) + rr;
    };
    auto load_state = [&](int cell) -> uint32_t {
        const int bit = cell * SB;
        return (stw[bit >> 5] >> (bit & 31)) & smask;
    };

    // ---- prologue: stage the stream, build (cos, sin) of the current phases ----------------
    if (IDX_SMEM) {
        uint2 *dst = reinterpret_cast<uint2 *>(smem_raw + L.idx);
        for (int q = tid; q < a.n_groups; q += NT) dst[q] = a.idx4[q];
    }
    for (int q = tid; q < n * RT; q += NT) {
        T s, c;
        phase_trig(phi[q], s, c);
        T2 v; v.x = c; v.y = s;
        cs[q] = v;
    }
    if (tid < RT) {
        T2 zero; zero.x = T(0); zero.y = T(0);
        cs[n * RT + tid] = zero;                  // dummy neighbour used by list padding
        best_s[tid] = a.best_obj[tile * RT + tid];
        improved_s[tid] = 0;
    }
    if (tid == 0) ks_s[a.step_begin & 1] = ks_value(a.ks_max, a.ks_period, (double)a.step_begin * a.h);
    __syncthreads();

    int sample_cur = 0;     // cursor into sample_steps
    while (sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] < a.step_begin) ++sample_cur;

    // score the state currently in cs/phi; sample_col >= 0 also records that trace column
    auto score_current = [&](long long step_label, int sample_col) {
        // 1. lattice states of own rows, packed SB bits per cell, one word per 32/SB lanes
        {
            int it = 0;
            for (int qd = slot; qd < ((quads + nslots - 1) / nslots) * nslots; qd += nslots, ++it) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = 4 * qd + k;
                    uint32_t s = 0;
                    if (i < n) s = (uint32_t)threshold_state((double)phi[i * RT + r], a.tc.n_states);
                    const int cell = ((it * 4 + k) << log2NT) + tid;
                    uint32_t v = s << ((cell * SB) & 31);
                    for (int off = 1; off < lanes_per_word; off <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, off);
                    if ((tid & (lanes_per_word - 1)) == 0) stw[(cell * SB) >> 5] = v;
                }
            }
        }
        __syncthreads();
        // 2. objective (and energy) over own rows, neighbours j > i only (canonical pairs)
        double obj_part = 0.0, en_part = 0.0;
        int g = g_start;
        for (int qd = slot; qd < quads; qd += nslots) {
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * qd + k;
                if (i >= n) break;
                const uint32_t si = load_state(state_cell(i, r));
                const T2 own = cs[i * RT + r];
                uint32_t last;
                do {
                    const uint2 pk = idx4[g];
                    last = pk.x & 0x8000u;
                    const int jj[4] = {(int)(pk.x & 0x7fffu), (int)(pk.x >> 16), (int)(pk.y & 0xffffu), (int)(pk.y >> 16)};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = jj[u];
                        if (j > i && j < n) {
                            const double w = WEIGHTED ? (double)wstream[4 * g + u] : 1.0;
                            const bool same = load_state(state_cell(j, r)) == si;
                            if (a.maximize) { if (!same) obj_part += w; }
                            else            { if (same) obj_part += 1.0; }
                            if (sample_col >= 0) {
                                const T2 v = cs[j * RT + r];
                                en_part += w * ((double)own.x * (double)v.x + (double)own.y * (double)v.y);
                            }
                        }
                    }
                    ++g;
                } while (!last);
            }
        }
        const double obj = tile_reduce(obj_part, RT, part, tid, nwarps);
        if (tid < RT) {
            const double b = best_s[tid];
            const bool better = a.maximize ? (obj > b) : (obj < b);
            improved_s[tid] = better ? 1 : 0;
            if (better) {
                best_s[tid] = obj;
                const int gi = tile * RT + tid;
                if (a.use_target && a.first_hit[gi] < 0 &&
                    (a.maximize ? (obj >= a.target) : (obj <= a.target)))
                    a.first_hit[gi] = step_label;
            }
        }
        __syncthreads();
        // 3. strict improvement: publish this replica's states
        if (improved_s[r] && live) {
            uint8_t *dst = a.best_states + (size_t)rg * n;
            for (int qd = slot; qd < quads; qd += nslots) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = 4 * qd + k;
                    if (i < n) dst[i] = (uint8_t)load_state(state_cell(i, r));
                }
            }
        }
        if (sample_col >= 0) {
            const double en = tile_reduce(en_part, RT, part, tid, nwarps);
            if (tid < RT) {
                const size_t gi = (size_t)(tile * RT + tid);
                a.energy[gi * a.trace_stride + sample_col] = en;
                a.best_trace[gi * a.trace_stride + sample_col] = best_s[tid];
            }
        }
        __syncthreads();
    };

    if (a.initial_sample) score_current(-1, 0);

    // ---- time loop ---------------------------------------------------------------------------
#pragma unroll 1
    for (long long step = a.step_begin; step < a.step_end; ++step) {
        const double ks = ks_s[step & 1];
        int g = g_start;
        // pass A: gather + update
#pragma unroll 1
        for (int qd = slot; qd < quads; qd += nslots) {
            T z[4] = {T(0), T(0), T(0), T(0)};
            if (a.noise_mode == 0) normals4(noise_block(seed, (uint64_t)step, (uint32_t)qd), z);
#pragma unroll 1
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * qd + k;
                if (i >= n) break;
                const T p = phi[i * RT + r];
                const T2 own = cs[i * RT + r];
                const T ci = own.x, si = own.y;
                T acc;
                uint32_t last;
                if (STRICT) {
                    acc = T(0);
                    do {
                        const uint2 pk = idx4[g];
                        last = pk.x & 0x8000u;
                        const int jj[4] = {(int)(pk.x & 0x7fffu), (int)(pk.x >> 16), (int)(pk.y & 0xffffu), (int)(pk.y >> 16)};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const T2 v = cs[jj[u] * RT + r];
                            const double w = WEIGHTED ? (double)wstream[4 * g + u] : 1.0;
                            const double term = __dsub_rn(__dmul_rn((double)si, (double)v.x), __dmul_rn((double)ci, (double)v.y));
                            acc = (T)__dadd_rn((double)acc, __dmul_rn(w, term));
                        }
                        ++g;
                    } while (!last);
                } else {
                    T ac = T(0), as = T(0);
                    do {
                        const uint2 pk = idx4[g];
                        last = pk.x & 0x8000u;
                        const T2 v0 = cs[(int)(pk.x & 0x7fffu) * RT + r];
                        const T2 v1 = cs[(int)(pk.x >> 16) * RT + r];
                        const T2 v2 = cs[(int)(pk.y & 0xffffu) * RT + r];
                        const T2 v3 = cs[(int)(pk.y >> 16) * RT + r];
                        if (WEIGHTED) {
                            const T w0 = wstream[4 * g], w1 = wstream[4 * g + 1], w2 = wstream[4 * g + 2], w3 = wstream[4 * g + 3];
                            ac = fma(w0, v0.x, ac); as = fma(w0, v0.y, as);
                            ac = fma(w1, v1.x, ac); as = fma(w1, v1.y, as);
                            ac = fma(w2, v2.x, ac); as = fma(w2, v2.y, as);
                            ac = fma(w3, v3.x, ac); as = fma(w3, v3.y, as);
                        } else {
                            ac += (v0.x + v1.x) + (v2.x + v3.x);
                            as += (v0.y + v1.y) + (v2.y + v3.y);
                        }
                        ++g;
                    } while (!last);
                    acc = si * ac - ci * as;
                }
                const T shil = shil_term(p, si, ci, a.tc);
                T kick = z[k];
                if (a.noise_mode == 1)
                    kick = live ? (T)a.noise_host[((size_t)(step - a.noise_step0) * a.R_real + rg) * n + i] : T(0);
                T x;
                if (STRICT) {
                    const double drift = __dsub_rn(__dmul_rn(a.K, (double)acc), __dmul_rn(ks, (double)shil));
                    x = (T)__dadd_rn(__dadd_rn((double)p, __dmul_rn(a.h, drift)), __dmul_rn(a.kn_sqrt_h, (double)kick));
                } else {
                    x = p + (T)a.h * ((T)a.K * acc - (T)ks * shil) + (T)a.kn_sqrt_h * kick;
                }
                if (!isfinite(x) && live) flag_nonfinite(a.nonfinite, (uint64_t)step, (uint32_t)rg, (uint32_t)i);
                phi[i * RT + r] = wrap_unit(x);
            }
        }
        if (tid == 0) ks_s[(step + 1) & 1] = ks_value(a.ks_max, a.ks_period, (double)(step + 1) * a.h);
        __syncthreads();
        // pass B: new (cos, sin)
#pragma unroll 1
        for (int qd = slot; qd < quads; qd += nslots) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * qd + k;
                if (i < n) {
                    T s, c;
                    phase_trig(phi[i * RT + r], s, c);
                    T2 v; v.x = c; v.y = s;
                    cs[i * RT + r] = v;
                }
            }
        }
        __syncthreads();
        // scoring schedule (dynamics.py:404-410)
        const bool is_sample = sample_cur < a.n_sample_steps && a.sample_steps[sample_cur] == step;
        if (is_sample) {
            score_current(step, a.sample_offset + sample_cur);
            ++sample_cur;
        } else if (a.cadence > 0 && step % a.cadence == 0) {
            score_current(step, -1);
        }
    }
    if (tid < RT) a.best_obj[tile * RT + tid] = best_s[tid];
}

} // namespace oscb
