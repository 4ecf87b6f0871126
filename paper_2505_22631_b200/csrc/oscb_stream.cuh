// oscb_stream.cuh -- "streaming" kernels: one launch per Euler step, phases and their
// (cos, sin) pairs live in HBM/L2 in the oscillator-major, replica-minor layout
//     X[i * R + r]          (i = oscillator, r = replica)
// so that the 32 lanes of a warp (consecutive r for R >= 32, consecutive i for R = 1) read a
// contiguous 128/256-byte segment for every neighbour gather -- the CSR SpMM over R batched
// replicas of north_star (2).  This path has no size limit; it is the general fallback, the
// single-step entry point (oscb_step == euler_step, dynamics.py:286-314), and the on-GPU
// cross-check of the resident kernel.
#pragma once
#include "oscb_device.cuh"

namespace oscb {

struct CsrDev {
    int n;
    const int *indptr;   // [n+1]
    const int *indices;  // [nnz]
    const double *w64;   // [nnz]
    const float *w32;    // [nnz]
};

template <typename T> __device__ __forceinline__ const T *csr_weights(const CsrDev &g);
template <> __device__ __forceinline__ const double *csr_weights<double>(const CsrDev &g) { return g.w64; }
template <> __device__ __forceinline__ const float *csr_weights<float>(const CsrDev &g) { return g.w32; }

// host layout [R, n] float64  <->  device layout [n, R] T
template <typename T>
__global__ void k_to_dev_layout(const double *__restrict__ src, T *__restrict__ dst, int n, int R)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n * R) return;
    const int i = (int)(q / R), r = (int)(q - (long long)i * R);
    dst[q] = (T)src[(long long)r * n + i];
}
template <typename T>
__global__ void k_from_dev_layout(const T *__restrict__ src, double *__restrict__ dst, int n, int R)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n * R) return;
    const int r = (int)(q / n), i = (int)(q - (long long)r * n);
    dst[q] = (double)src[(long long)i * R + r];
}

// exact numpy Philox initial phases, written straight into the host layout [R, n] float64
__global__ void k_initial_phases(const uint64_t *__restrict__ seeds, double *__restrict__ phi, int n, int R)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int quads = (n + 3) >> 2;
    if (q >= (long long)quads * R) return;
    const int r = (int)(q / quads), quad = (int)(q - (long long)r * quads);
    uint64_t w[4];
    // counter (1 << 192) pre-incremented before every block: low word = 1 + quad
    philox4x64_10(1ull + (uint64_t)quad, 0ull, 0ull, 1ull, seeds[r], 0ull, w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int i = 4 * quad + k;
        if (i < n) phi[(long long)r * n + i] = (double)(w[k] >> 11) * (1.0 / 9007199254740992.0);
    }
}

// the integrator's own normals for (seed, step, oscillators 0..n-1), widened to float64
template <typename T>
__global__ void k_device_normals(uint64_t seed, uint64_t step, int n, double *__restrict__ out)
{
    const int quad = blockIdx.x * blockDim.x + threadIdx.x;
    if (quad >= (n + 3) / 4) return;
    T z[4];
    normals4(noise_block(seed, step, (uint32_t)quad), z);
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (4 * quad + k < n) out[4 * quad + k] = (double)z[k];
}

// (cos, sin) of every phase: cs[i*R + r] = {cos 2pi phi, sin 2pi phi}
template <typename T>
__global__ void k_trig(const T *__restrict__ phi, typename Vec2<T>::type *__restrict__ cs, long long total)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= total) return;
    T s, c;
    phase_trig(phi[q], s, c);
    typename Vec2<T>::type v; v.x = c; v.y = s;
    cs[q] = v;
}

struct StepScalars {
    double K, ks, h, kn_sqrt_h;
    TrigConst tc;
    uint64_t step;      // global step index (noise counter, non-finite report)
    int noise_mode;     // OSCB_NOISE_*
};

// One Euler step.  A thread owns one replica r and the four consecutive oscillators of one
// quad (one Philox block = four normals).  STRICT (fp64 parity mode) keeps the reference's
// operation order: per-term acc += w*(s_i*c_j - c_i*s_j) in CSR order with no contraction.
template <typename T, bool STRICT>
__global__ void __launch_bounds__(256)
k_stream_step(CsrDev g, int R, const T *__restrict__ phi_in,
              const typename Vec2<T>::type *__restrict__ cs_in, T *__restrict__ phi_out,
              typename Vec2<T>::type *__restrict__ cs_out, const uint64_t *__restrict__ seeds,
              const double *__restrict__ noise_host /* [R, n] or null */, StepScalars sc,
              unsigned long long *__restrict__ nonfinite)
{
    using T2 = typename Vec2<T>::type;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int quads = (g.n + 3) >> 2;
    if (q >= (long long)quads * R) return;
    const int quad = (int)(q / R), r = (int)(q - (long long)quad * R);
    const T *__restrict__ wt = csr_weights<T>(g);

    T z[4] = {T(0), T(0), T(0), T(0)};
    if (sc.noise_mode == 0) normals4(noise_block(seeds[r], sc.step, (uint32_t)quad), z);

#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
        const int i = 4 * quad + k;
        if (i >= g.n) break;
        const long long me = (long long)i * R + r;
        const T2 own = cs_in[me];
        const T ci = own.x, si = own.y;
        const int beg = g.indptr[i], end = g.indptr[i + 1];
        T acc;
        if (STRICT) {
            acc = T(0);
            for (int e = beg; e < end; ++e) {
                const T2 v = cs_in[(long long)g.indices[e] * R + r];
                const double term = __dsub_rn(__dmul_rn((double)si, (double)v.x), __dmul_rn((double)ci, (double)v.y));
                acc = (T)__dadd_rn((double)acc, __dmul_rn((double)wt[e], term));
            }
        } else {
            T ac = T(0), as = T(0);
            for (int e = beg; e < end; ++e) {
                const T2 v = cs_in[(long long)g.indices[e] * R + r];
                const T w = wt[e];
                ac = fma(w, v.x, ac);
                as = fma(w, v.y, as);
            }
            acc = si * ac - ci * as;
        }
        const T p = phi_in[me];
        const T shil = shil_term(p, si, ci, sc.tc);
        T kick;
        if (sc.noise_mode == 1) kick = (T)noise_host[(long long)r * g.n + i];
        else kick = z[k];
        T x;
        if (STRICT) {
            const double drift = __dsub_rn(__dmul_rn(sc.K, (double)acc), __dmul_rn(sc.ks, (double)shil));
            x = (T)__dadd_rn(__dadd_rn((double)p, __dmul_rn(sc.h, drift)), __dmul_rn(sc.kn_sqrt_h, (double)kick));
        } else {
            x = p + (T)sc.h * ((T)sc.K * acc - (T)sc.ks * shil) + (T)sc.kn_sqrt_h * kick;
        }
        if (!isfinite(x)) flag_nonfinite(nonfinite, sc.step, (uint32_t)r, (uint32_t)i);
        const T y = wrap_unit(x);
        phi_out[me] = y;
        T s2, c2;
        phase_trig(y, s2, c2);
        T2 o; o.x = c2; o.y = s2;
        cs_out[me] = o;
    }
}

// threshold every phase to its lattice state (device layout in, device layout out)
template <typename T>
__global__ void k_threshold(const T *__restrict__ phi, uint8_t *__restrict__ states, long long total, int n_states)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= total) return;
    states[q] = (uint8_t)threshold_state((double)phi[q], n_states);
}

// fixed-order block reduction (deterministic): shuffle tree inside a warp, then warp 0 sums
// the per-warp partials in index order.
__device__ __forceinline__ double block_sum_256(double v, double *scratch /* [8] */)
{
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double tot = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += scratch[w];
    return tot; // valid in thread 0
}

// objective per replica over the canonical pairs (dynamics.py:214-223), replica index on the
// lanes so every state read is a coalesced 32-byte segment of the [n, R] layout.
// grid = (ceil(R/32), P): block (x, p) covers replicas 32x..32x+31 and the p-th chunk of pairs;
// its 8 warps stride through the chunk.  partial[p * R + r] is summed in index order by
// k_best_flag, so the result does not depend on scheduling.
// maximize: sum w [s_u != s_v];  else: count [s_u == s_v].
__global__ void __launch_bounds__(256)
k_objective_partial(const uint8_t *__restrict__ states, int R, const int *__restrict__ iu,
                    const int *__restrict__ jv, const double *__restrict__ w, int m, int chunk,
                    int maximize, double *__restrict__ partial)
{
    __shared__ double part[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = blockIdx.x * 32 + lane;
    const int e0 = blockIdx.y * chunk, e1 = min(m, e0 + chunk);
    double acc = 0.0;
    if (r < R) {
        for (int e = e0 + warp; e < e1; e += 8) {
            const bool same = states[(long long)iu[e] * R + r] == states[(long long)jv[e] * R + r];
            if (maximize) { if (!same) acc += w[e]; }
            else          { if (same) acc += 1.0; }
        }
    }
    part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && r < R) {
        double tot = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) tot += part[k][lane];
        partial[(long long)blockIdx.y * R + r] = tot;
    }
}

// the reference's own summation order (one thread walks all pairs of one replica): used by
// oscb_score when the couplings are not integer valued, where the order is visible in the
// last bits of the sum.
__global__ void k_objective_seq(const uint8_t *__restrict__ states, int R, const int *__restrict__ iu,
                                const int *__restrict__ jv, const double *__restrict__ w, int m,
                                int maximize, double *__restrict__ obj)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    double acc = 0.0;
    for (int e = 0; e < m; ++e) {
        const bool same = states[(long long)iu[e] * R + r] == states[(long long)jv[e] * R + r];
        if (maximize) { if (!same) acc = __dadd_rn(acc, w[e]); }
        else          { if (same) acc += 1.0; }
    }
    obj[r] = acc;
}

// continuous energy per replica (dynamics.py:380): sum_e w_e cos(2 pi (phi_u - phi_v))
template <typename T>
__global__ void __launch_bounds__(256)
k_energy(const T *__restrict__ phi, int R, const int *__restrict__ iu, const int *__restrict__ jv,
         const double *__restrict__ w, int m, double *__restrict__ out, long long out_stride)
{
    __shared__ double scratch[8];
    const int r = blockIdx.x;
    double part = 0.0;
    for (int e = threadIdx.x; e < m; e += blockDim.x) {
        const double d = (double)phi[(long long)iu[e] * R + r] - (double)phi[(long long)jv[e] * R + r];
        part += w[e] * cos(__dmul_rn(OSCB_TWO_PI, d));
    }
    const double tot = block_sum_256(part, scratch);
    if (threadIdx.x == 0) out[(long long)r * out_stride] = tot;
}

// best-so-far bookkeeping (dynamics.py:370-375): strict improvement only.  obj[r] is the
// in-order sum of the P partials of k_objective_partial (P == 1: obj already final).
__global__ void k_best_flag(const double *__restrict__ partial, int P, double *__restrict__ obj,
                            double *__restrict__ best_obj, uint8_t *__restrict__ improved,
                            long long *__restrict__ first_hit, int R, int maximize, int use_target,
                            double target, long long step)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    double o = 0.0;
    for (int p = 0; p < P; ++p) o += partial[(long long)p * R + r];
    obj[r] = o;
    if (!best_obj) return;
    const double b = best_obj[r];
    const bool better = maximize ? (o > b) : (o < b);
    improved[r] = better ? 1 : 0;
    if (better) {
        best_obj[r] = o;
        if (use_target && first_hit[r] < 0 && (maximize ? (o >= target) : (o <= target))) first_hit[r] = step;
    }
}
// states: device layout [n, R]; best_states: host layout [R, n]
__global__ void k_best_copy(const uint8_t *__restrict__ states, const uint8_t *__restrict__ improved,
                            uint8_t *__restrict__ best_states, int n, int R)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n * R) return;
    const int i = (int)(q / R), r = (int)(q - (long long)i * R);
    if (improved[r]) best_states[(long long)r * n + i] = states[q];
}
__global__ void k_record_best(const double *__restrict__ best_obj, double *__restrict__ best_trace,
                              long long stride, int R)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < R) best_trace[(long long)r * stride] = best_obj[r];
}
// transposed state copy for oscb_score: [n, R] u8 -> [R, n] int64
__global__ void k_states_to_host_layout(const uint8_t *__restrict__ states, long long *__restrict__ out, int n, int R)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n * R) return;
    const int r = (int)(q / n), i = (int)(q - (long long)r * n);
    out[q] = states[(long long)i * R + r];
}

} // namespace oscb
