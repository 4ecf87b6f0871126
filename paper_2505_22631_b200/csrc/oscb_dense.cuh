// oscb_dense.cuh -- dense all-to-all couplings (SK-type graphs): the Euler step as a row-tiled
// J * [cos Theta | sin Theta] product with the SHIL / noise / wrap epilogue fused in, and the
// matching O(n^2) scoring / energy kernels.  One handle holds a ROW SHARD J[row_begin:row_end, :]
// (the whole matrix on one GPU, or 1/G of it per rank with the phases all-gathered every step,
// SURVEY.md 8e).
//
// Layouts: J shard row-major [rows][n] in JT (int8 when every coupling is an integer in
// [-127, 127] -- +-1 SK couplings cost 1 byte of HBM per update -- else float32 / float64);
// phases and (cos, sin) pairs oscillator-major, replica-minor [n][R] like the streaming kernels.
//
// A warp owns one row at a time and RB replicas of it: the 32 lanes stride over the columns, each
// J entry is loaded once and applied to the RB replicas' pairs, the lanes' partial sums are
// combined with a shuffle tree, and lanes 0..RB-1 run the epilogue of one replica each.
// R = 1 is a GEMV bound by the HBM read of J; for many replicas this SIMT form is compute bound.
// Integer couplings with N = 2 run on the tensor-core kernel instead (oscb_umma.cuh); this is the
// general dense path (any weights, any N, host-injected noise) and the single-step entry point.  Summation order is a fixed tree, not the
// reference's sequential CSR order, so dense float64 parity is to rounding (~1e-13), not bitwise.
//
// Reference arithmetic restated: dynamics.py:166-172 (row update), :214-223 (objectives),
// :380 (energy).
#pragma once
#include "oscb_device.cuh"
#include "oscb_stream.cuh"

namespace oscb {

template <typename JT> struct JVec;      // vector load of 4 couplings (2 for double)
template <> struct JVec<int8_t> {
    static constexpr int N = 4;
    __device__ static void load(const int8_t *p, float (&w)[4])
    {
        const char4 v = *reinterpret_cast<const char4 *>(p);
        w[0] = (float)v.x; w[1] = (float)v.y; w[2] = (float)v.z; w[3] = (float)v.w;
    }
    __device__ static void load(const int8_t *p, double (&w)[4])
    {
        const char4 v = *reinterpret_cast<const char4 *>(p);
        w[0] = (double)v.x; w[1] = (double)v.y; w[2] = (double)v.z; w[3] = (double)v.w;
    }
};
template <> struct JVec<float> {
    static constexpr int N = 4;
    __device__ static void load(const float *p, float (&w)[4])
    {
        const float4 v = *reinterpret_cast<const float4 *>(p);
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    }
    __device__ static void load(const float *p, double (&w)[4])
    {
        const float4 v = *reinterpret_cast<const float4 *>(p);
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    }
};
template <> struct JVec<double> {
    static constexpr int N = 4;
    __device__ static void load(const double *p, float (&w)[4])
    {
        const double2 a = *reinterpret_cast<const double2 *>(p), b = *reinterpret_cast<const double2 *>(p + 2);
        w[0] = (float)a.x; w[1] = (float)a.y; w[2] = (float)b.x; w[3] = (float)b.y;
    }
    __device__ static void load(const double *p, double (&w)[4])
    {
        const double2 a = *reinterpret_cast<const double2 *>(p), b = *reinterpret_cast<const double2 *>(p + 2);
        w[0] = a.x; w[1] = a.y; w[2] = b.x; w[3] = b.y;
    }
};

struct DenseStepArgs {
    int n;                 // oscillators (columns of J); n % 4 == 0 is arranged by padding J on upload
    int n_pad;             // row stride of J in elements (multiple of 4)
    int row_begin, rows;   // this shard's rows [row_begin, row_begin + rows)
    int R;
    StepScalars sc;
};

// One Euler step of the shard's rows.  phi_in / cs_in: all n oscillators [n][R]; phi_out, cs_out:
// rows of this shard only, [rows][R] (cs_out may be null: the sharded driver rebuilds the pairs
// from the gathered phases).  Grid: (ceil(rows / 8), ceil(R / RB)), 256 threads.
template <typename T, typename JT, int RB>
__global__ void __launch_bounds__(256)
k_dense_step(DenseStepArgs a, const JT *__restrict__ J, const T *__restrict__ phi_in,
             const typename Vec2<T>::type *__restrict__ cs_in, T *__restrict__ phi_out,
             typename Vec2<T>::type *__restrict__ cs_out, const uint64_t *__restrict__ seeds,
             const double *__restrict__ noise_host /* [R, n] or null */, unsigned long long *__restrict__ nonfinite)
{
    using T2 = typename Vec2<T>::type;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row_local = blockIdx.x * 8 + warp;
    if (row_local >= a.rows) return;
    const int i = a.row_begin + row_local;
    const int r0 = blockIdx.y * RB;
    const int R = a.R;
    T2 acc[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) { acc[r].x = T(0); acc[r].y = T(0); }
    const JT *Jrow = J + (size_t)row_local * a.n_pad;
    for (int j0 = lane * 4; j0 < a.n; j0 += 128) {
        T w[4];
        JVec<JT>::load(Jrow + j0, w);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int j = j0 + v;
            if (j < a.n) {
                const T2 *src = cs_in + (size_t)j * R + r0;
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                    if (RB == 1 || r0 + r < R) {
                        const T2 c = src[r];
                        acc[r].x = fma(w[v], c.x, acc[r].x);
                        acc[r].y = fma(w[v], c.y, acc[r].y);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r)
        for (int off = 16; off > 0; off >>= 1) {
            acc[r].x += __shfl_xor_sync(0xffffffffu, acc[r].x, off);
            acc[r].y += __shfl_xor_sync(0xffffffffu, acc[r].y, off);
        }
    // lanes 0..RB-1: epilogue of replica r0 + lane
    T2 mine = acc[0];
#pragma unroll
    for (int r = 1; r < RB; ++r)
        if (lane == r) mine = acc[r];
    const int rr = r0 + lane;
    if (lane < RB && rr < R) {
        const size_t me = (size_t)i * R + rr;
        const T2 own = cs_in[me];
        const T ci = own.x, si = own.y;
        const T p = phi_in[me];
        const T accv = si * mine.x - ci * mine.y;
        const T shil = shil_term(p, si, ci, a.sc.tc);
        T kick = T(0);
        if (a.sc.noise_mode == 0) {
            T z[4];
            normals4(noise_block(seeds[rr], a.sc.step, (uint32_t)(i >> 2)), z);
            kick = z[i & 3];
        } else if (a.sc.noise_mode == 1) {
            kick = (T)noise_host[(size_t)rr * a.n + i];
        }
        const T x = p + (T)a.sc.h * ((T)a.sc.K * accv - (T)a.sc.ks * shil) + (T)a.sc.kn_sqrt_h * kick;
        if (!isfinite(x)) flag_nonfinite(nonfinite, a.sc.step, (uint32_t)rr, (uint32_t)i);
        const T y = wrap_unit(x);
        const size_t out = (size_t)row_local * R + rr;
        phi_out[out] = y;
        if (cs_out) {
            T s2, c2;
            phase_trig(y, s2, c2);
            T2 o; o.x = c2; o.y = s2;
            cs_out[out] = o;
        }
    }
}

// Per-row partial objectives / energies of the shard's rows over the columns j > i (canonical
// pairs): MODE 0 = cut weight sum J_ij [s_i != s_j]; 1 = conflicts [J_ij != 0][s_i == s_j];
// 2 = energy sum J_ij (c_i c_j + s_i s_j).  partial: [rows][R] (summed in row order by
// k_dense_reduce, so the result does not depend on scheduling).
template <typename T, typename JT, int MODE>
__global__ void __launch_bounds__(256)
k_dense_pairs(int n, int n_pad, int row_begin, int rows, int R, const JT *__restrict__ J,
              const uint8_t *__restrict__ states /* [n][R], MODE 0/1 */,
              const typename Vec2<T>::type *__restrict__ cs /* [n][R], MODE 2 */, double *__restrict__ partial)
{
    using T2 = typename Vec2<T>::type;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row_local = blockIdx.x * 8 + warp;
    if (row_local >= rows) return;
    const int i = row_begin + row_local;
    const int r = blockIdx.y;
    const JT *Jrow = J + (size_t)row_local * n_pad;
    double acc = 0.0;
    uint8_t si = 0;
    T2 own; own.x = T(0); own.y = T(0);
    if (MODE == 2) own = cs[(size_t)i * R + r];
    else si = states[(size_t)i * R + r];
    const int jstart = ((i + 1) / 4) * 4;              // first aligned group that can hold a j > i
    for (int j0 = jstart + lane * 4; j0 < n; j0 += 128) {
        double w[4];
        JVec<JT>::load(Jrow + j0, w);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int j = j0 + v;
            if (j > i && j < n && w[v] != 0.0) {
                if (MODE == 0) { if (states[(size_t)j * R + r] != si) acc += w[v]; }
                else if (MODE == 1) { if (states[(size_t)j * R + r] == si) acc += 1.0; }
                else {
                    const T2 c = cs[(size_t)j * R + r];
                    acc += w[v] * ((double)own.x * (double)c.x + (double)own.y * (double)c.y);
                }
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) partial[(size_t)row_local * R + r] = acc;
}

// obj[r] (+)= sum over the shard's rows, in row order.  One thread per replica.
__global__ void k_dense_reduce(const double *__restrict__ partial, int rows, int R, double *__restrict__ out, long long out_stride)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    double tot = 0.0;
    for (int q = 0; q < rows; ++q) tot += partial[(size_t)q * R + r];
    out[(long long)r * out_stride] = tot;
}

// gather rows [row_begin, row_begin + rows) of a full [n][R] array (used to seed a shard's slice)
template <typename T>
__global__ void k_dense_copy_rows(const T *__restrict__ full, T *__restrict__ rows_out, int row_begin, int rows, int R)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)rows * R) return;
    rows_out[q] = full[(long long)row_begin * R + q];
}

} // namespace oscb
