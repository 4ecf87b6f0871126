// oscb_csr_build.cu -- device-side build of the symmetric CSR from an edge list: the GPU form of
// CouplingMatrix.from_edges (reference model.py:151-200).  One (i, j, x) entry per unordered pair in, the canonical CSR
// out (both directions, rows ascending, columns ascending inside a row, entries with x == 0 dropped) -- the same arrays,
// bit for bit, as the vectorised host build in model.py, with the reference's validation in the reference's order
// (index range, then self-coupling, then a pair listed twice -- zero-valued entries included, as the reference checks
// before it filters).
//
// Integer / byte work, HBM-bound, no sort of the whole list:
//   k_csr_count        degree histogram with atomics + range / diagonal / has-zero flags        24 B read per entry
//   k_csr_scan         exclusive scan of the degrees -> indptr (block totals | scan of the totals | prefixes; n words)
//   k_csr_fill         scatter both directions into the rows in arrival order, 16 B per entry    24 B read, 32 B written
//   k_csr_sort_short   rows of <= 32 entries: a warp per batch of rows, rank by counting (shuffles) 16 B read, 16 B written per entry
//   k_csr_sort_long    longer rows, a CTA per row.  Columns of a row are unique, so the position of column c is the number
//                      of set bits below c in the row's column BITMAP (n bits in shared memory, a popcount prefix per 1024
//                      columns): O(n / 32 + d) per row, and a bit found set twice is the duplicate pair.  Rows too short to
//                      pay for clearing the bitmap (or n beyond shared memory) rank by counting, O(d^2 / threads).
//   k_csr_compact      only when some x == 0: per-row stable compaction to the final arrays
#include "oscb_host.hpp"

#include <algorithm>
#include <exception>

namespace oscb {

constexpr uint32_t CSR_ERANGE = 1u, CSR_EDIAG = 2u, CSR_EDUP = 4u, CSR_HASZERO = 8u;
constexpr int CSR_LONG_THREADS = 512;

__global__ void __launch_bounds__(256) k_csr_count(int64_t m, int64_t n, const int64_t *__restrict__ ei, const int64_t *__restrict__ ej,
                                                   const double *__restrict__ ex, uint32_t *deg, uint32_t *flags)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += stride) {
        const int64_t e = base + threadIdx.x;
        uint32_t f = 0;
        if (e < m) {
            const int64_t a = ei[e], b = ej[e];
            if (a < 0 || b < 0 || a >= n || b >= n) f |= CSR_ERANGE;
            else if (a == b) f |= CSR_EDIAG;
            else {
                atomicAdd(&deg[a], 1u);
                atomicAdd(&deg[b], 1u);
            }
            if (ex[e] == 0.0) f |= CSR_HASZERO;
        }
        f = __reduce_or_sync(0xffffffffu, f);
        if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
    }
}

// the same histogram through a shared-memory copy of the counters (n <= CSR_SMEM_COUNTERS): on dense graphs every entry hits
// one of a few thousand counters and the global atomics queue up in L2 (complete graph on 4096 oscillators: 404 us -> see
// DESIGN 4d); a CTA counts privately and adds its non-zero counters once.
constexpr int CSR_SMEM_COUNTERS = 16384;
__global__ void __launch_bounds__(512) k_csr_count_smem(int64_t m, int64_t n, const int64_t *__restrict__ ei, const int64_t *__restrict__ ej,
                                                        const double *__restrict__ ex, uint32_t *deg, uint32_t *flags)
{
    extern __shared__ uint32_t csr_hist[];
    for (int k = threadIdx.x; k < (int)n; k += blockDim.x) csr_hist[k] = 0u;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += stride) {
        const int64_t e = base + threadIdx.x;
        uint32_t f = 0;
        if (e < m) {
            const int64_t a = ei[e], b = ej[e];
            if (a < 0 || b < 0 || a >= n || b >= n) f |= CSR_ERANGE;
            else if (a == b) f |= CSR_EDIAG;
            else {
                atomicAdd(&csr_hist[a], 1u);
                atomicAdd(&csr_hist[b], 1u);
            }
            if (ex[e] == 0.0) f |= CSR_HASZERO;
        }
        f = __reduce_or_sync(0xffffffffu, f);
        if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < (int)n; k += blockDim.x)
        if (csr_hist[k]) atomicAdd(&deg[k], csr_hist[k]);
}

// Exclusive scan in three launches of one kernel.  CTA b scans cnt[b * L, (b + 1) * L) in trips of 4096 entries (1024 threads x
// 4), starting from block_off[b] (0 when NULL); it writes the prefixes to out (skipped when NULL), its own total to tot[b]
// (skipped when NULL), and the CTA that reaches n writes out[n].  Pass 1: totals of 4096-entry blocks; pass 2: one CTA scans
// the totals; pass 3: the prefixes.  (One CTA walking the whole array took 0.78 ms at n = 10^6 -- 3.2 us per dependent trip --
// which was 60 % of the build.)
template <typename T>
__global__ void __launch_bounds__(1024) k_csr_scan(int64_t n, int64_t L, const T *__restrict__ cnt, int64_t *__restrict__ out,
                                                   const int64_t *__restrict__ block_off, unsigned long long *__restrict__ tot)
{
    __shared__ long long warp_tot[32];
    __shared__ long long trip_total;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t begin = (int64_t)blockIdx.x * L, end = begin + L < n ? begin + L : n;
    const long long start = block_off ? (long long)block_off[blockIdx.x] : 0;
    long long carry = start;
    for (int64_t base = begin; base < end; base += 4096) {
        const int64_t i0 = base + 4 * (int64_t)tid;
        long long d[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) d[k] = i0 + k < end ? (long long)cnt[i0 + k] : 0;
        const long long mine = (d[0] + d[1]) + (d[2] + d[3]);
        long long incl = mine;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const long long up = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += up;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const long long t = warp_tot[lane];
            long long s = t;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const long long up = __shfl_up_sync(0xffffffffu, s, off);
                if (lane >= off) s += up;
            }
            warp_tot[lane] = s - t;                       // exclusive prefix of the warps
        }
        __syncthreads();
        long long p = carry + warp_tot[warp] + (incl - mine);
        if (out) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (i0 + k < end) out[i0 + k] = p;
                p += d[k];
            }
        }
        if (tid == 1023) trip_total = warp_tot[31] + incl;     // prefix of the last warp + its inclusive sum
        __syncthreads();
        carry += trip_total;
        __syncthreads();
    }
    if (tid == 0) {
        if (tot) tot[blockIdx.x] = (unsigned long long)(carry - start);
        if (out && end == n && (begin < n || blockIdx.x == 0)) out[n] = carry;
    }
}

// both directions of every entry into its rows, in arrival order (the sort kernels put a row in column order).  `deg` counts
// down to zero: it is the cursor.  An entry travels as ONE 16-byte store {column, value bits}: a scattered store costs a 32-byte
// sector whatever its size, so column and value in separate arrays cost two.
__global__ void __launch_bounds__(256) k_csr_fill(int64_t m, const int64_t *__restrict__ ei, const int64_t *__restrict__ ej,
                                                  const double *__restrict__ ex, const int64_t *__restrict__ indptr, uint32_t *deg,
                                                  longlong2 *__restrict__ tent)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const int64_t a = ei[e], b = ej[e];
        const long long v = __double_as_longlong(ex[e]);
        const int64_t pa = indptr[a] + (int64_t)(atomicSub(&deg[a], 1u) - 1u);
        tent[pa] = make_longlong2(b, v);
        const int64_t pb = indptr[b] + (int64_t)(atomicSub(&deg[b], 1u) - 1u);
        tent[pb] = make_longlong2(a, v);
    }
}

// Rows of <= 32 entries.  A warp owns a contiguous block of rows and takes, per trip, as many consecutive rows as fit into its 32
// lanes (a low-degree graph: four to eight rows at once instead of one -- the kernel is a chain of dependent loads per trip, so
// trips are what it costs), a lane per entry; an entry's place = the number of smaller columns in its own row (shuffles over the
// batch, masked by the row's lane range); equal columns in a row = the duplicate pair.  A row of more than 32 entries goes on the
// list for k_csr_sort_long.
__global__ void __launch_bounds__(256) k_csr_sort_short(int64_t n, int64_t rows_per_warp, const int64_t *__restrict__ indptr,
                                                        const longlong2 *__restrict__ tent, int64_t *__restrict__ ocols,
                                                        double *__restrict__ ovals, int32_t *long_rows, uint32_t *n_long, uint32_t *flags)
{
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t begin = w * rows_per_warp, end = begin + rows_per_warp < n ? begin + rows_per_warp : n;
    for (int64_t row = begin; row < end;) {
        const int cand = (int)(end - row < 31 ? end - row : 31);                    // rows this trip may take
        const int64_t ip = lane <= cand ? indptr[row + lane] : 0;                    // lane l: start of row + l
        const int64_t base = __shfl_sync(0xffffffffu, ip, 0);
        const uint32_t fit = __ballot_sync(0xffffffffu, lane >= 1 && lane <= cand && ip - base <= 32);
        if (fit == 0u) {                                                             // the first row alone is too long
            if (lane == 0) long_rows[atomicAdd(n_long, 1u)] = (int32_t)row;
            row += 1;
            continue;
        }
        const int k = 31 - __clz(fit);                                               // rows [row, row + k) fit (prefixes are monotone)
        const int total = (int)(__shfl_sync(0xffffffffu, ip, k) - base);
        const bool mine = lane < total;
        longlong2 ent = make_longlong2(0x7fffffffffffffffll, 0);
        if (mine) ent = tent[base + lane];
        int seg = 0;                                                                 // my row = row + seg
        for (int r = 1; r < k; ++r) seg += (int)(__shfl_sync(0xffffffffu, ip, r) - base) <= lane;
        const int seg_lo = (int)(__shfl_sync(0xffffffffu, ip, seg) - base), seg_hi = (int)(__shfl_sync(0xffffffffu, ip, seg + 1) - base);
        // (columns are < 2^31: the shuffles carry 32 bits; "equal to my own column in my row" counts me once, hence the - 1)
        const int c32 = mine ? (int)ent.x : 0x7fffffff;
        int rank = 0, same = 0;
#pragma unroll 4
        for (int l = 0; l < total; ++l) {
            const int cl = __shfl_sync(0xffffffffu, c32, l);
            const bool inrow = (unsigned)(l - seg_lo) < (unsigned)(seg_hi - seg_lo);
            rank += inrow && cl < c32;
            same += inrow && cl == c32;
        }
        const bool dup = same > 1;
        if (mine) {
            if (dup) atomicOr(flags, CSR_EDUP);
            else {
                ocols[base + seg_lo + rank] = ent.x;
                ovals[base + seg_lo + rank] = __longlong_as_double(ent.y);
            }
        }
        row += k;
    }
}

// rows of more than 32 entries, one CTA per row (see the header of this file)
__global__ void __launch_bounds__(CSR_LONG_THREADS) k_csr_sort_long(int64_t n, int bitmap_fits, const int64_t *__restrict__ indptr,
                                                                    const longlong2 *__restrict__ tent,
                                                                    int64_t *__restrict__ ocols, double *__restrict__ ovals,
                                                                    const int32_t *__restrict__ long_rows, const uint32_t *__restrict__ n_long,
                                                                    uint32_t *flags)
{
    extern __shared__ uint32_t csr_sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t W = (uint32_t)((n + 31) >> 5), CH = (W + 31) >> 5;     // bitmap words; chunks of 32 words
    uint32_t *bitmap = csr_sm, *cpre = csr_sm + W;
    const uint32_t count = *n_long;
    for (uint32_t li = blockIdx.x; li < count; li += gridDim.x) {
        const int64_t row = long_rows[li];
        const int64_t lo = indptr[row];
        const int64_t d = indptr[row + 1] - lo;
        const longlong2 *re = tent + lo;
        bool dup = false;
        if (bitmap_fits && d * d > (n >> 3) + 32 * d) {
            for (uint32_t w = tid; w < W; w += CSR_LONG_THREADS) bitmap[w] = 0u;
            __syncthreads();
            for (int64_t e = tid; e < d; e += CSR_LONG_THREADS) {
                const uint32_t c = (uint32_t)re[e].x, bit = 1u << (c & 31);
                dup = dup || (atomicOr(&bitmap[c >> 5], bit) & bit);
            }
            __syncthreads();
            for (uint32_t ch = warp; ch < CH; ch += CSR_LONG_THREADS / 32) {
                const uint32_t w = ch * 32 + lane;
                const uint32_t tot = __reduce_add_sync(0xffffffffu, w < W ? (uint32_t)__popc(bitmap[w]) : 0u);
                if (lane == 0) cpre[ch] = tot;
            }
            __syncthreads();
            if (warp == 0) {
                uint32_t carry = 0;
                for (uint32_t base = 0; base < CH; base += 32) {
                    const uint32_t t = base + lane < CH ? cpre[base + lane] : 0u;
                    uint32_t s = t;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const uint32_t up = __shfl_up_sync(0xffffffffu, s, off);
                        if (lane >= off) s += up;
                    }
                    if (base + lane < CH) cpre[base + lane] = carry + s - t;
                    carry += __shfl_sync(0xffffffffu, s, 31);
                }
            }
            __syncthreads();
            if (!__syncthreads_or(dup)) {
                for (int64_t e = tid; e < d; e += CSR_LONG_THREADS) {
                    const longlong2 ent = re[e];
                    const uint32_t c = (uint32_t)ent.x, wd = c >> 5, ch = wd >> 5;
                    uint32_t rank = cpre[ch];
                    for (uint32_t w = ch * 32; w < wd; ++w) rank += __popc(bitmap[w]);
                    rank += __popc(bitmap[wd] & ((1u << (c & 31)) - 1u));
                    ocols[lo + rank] = (int64_t)c;
                    ovals[lo + rank] = __longlong_as_double(ent.y);
                }
            }
            __syncthreads();
        } else {
            for (int64_t e = tid; e < d; e += CSR_LONG_THREADS) {
                const longlong2 ent = re[e];
                const long long c = ent.x;
                int64_t rank = 0;
                bool twice = false;
                for (int64_t f = 0; f < d; ++f) {
                    const long long cf = re[f].x;
                    rank += cf < c;
                    twice = twice || (cf == c && f != e);
                }
                if (twice) dup = true;
                else {
                    ocols[lo + rank] = c;
                    ovals[lo + rank] = __longlong_as_double(ent.y);
                }
            }
        }
        if (dup) atomicOr(flags, CSR_EDUP);
    }
}

// entries of a row with x != 0 (reference model.py:178: the filter comes after the validation)
__global__ void __launch_bounds__(256) k_csr_nzcount(int64_t n, const int64_t *__restrict__ indptr, const double *__restrict__ vals, uint32_t *cnt)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
        const int64_t lo = indptr[row], hi = indptr[row + 1];
        uint32_t c = 0;
        for (int64_t e = lo + lane; e < hi; e += 32) c += vals[e] != 0.0;
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) cnt[row] = c;
    }
}

__global__ void __launch_bounds__(256) k_csr_compact(int64_t n, const int64_t *__restrict__ indptr, const int64_t *__restrict__ indptr2,
                                                     const int64_t *__restrict__ cols, const double *__restrict__ vals,
                                                     int64_t *__restrict__ ccols, double *__restrict__ cvals)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
        const int64_t lo = indptr[row], hi = indptr[row + 1];
        int64_t dst = indptr2[row];
        for (int64_t base = lo; base < hi; base += 32) {
            const int64_t e = base + lane;
            const double v = e < hi ? vals[e] : 0.0;
            const bool keep = e < hi && v != 0.0;
            const uint32_t mask = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int64_t p = dst + __popc(mask & ((1u << lane) - 1u));
                ccols[p] = cols[e];
                cvals[p] = v;
            }
            dst += __popc(mask);
        }
    }
}

namespace {
// Scratch of a build.  Small builds (<= 512 MB in total) take their blocks from the run-time pool (cudaMalloc + cudaFree of a
// dozen blocks is 5-8 ms, as much as the rest of a 2 x 10^6-edge call); a large one uses plain cudaMalloc blocks and gives them
// back, so that a one-off build of a large graph does not park gigabytes in the pool.
template <typename T> struct Scratch {
    T *p = nullptr;
    size_t bytes = 0;
    bool pooled = false;
    Scratch(size_t count, bool use_pool) : bytes((count ? count : 1) * sizeof(T)), pooled(use_pool)
    {
        if (pooled) p = static_cast<T *>(pool_alloc(bytes));
        else OSCB_CUDA(cudaMalloc(&p, bytes));
    }
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    ~Scratch()
    {
        if (!p) return;
        if (pooled) pool_free(p, bytes);
        else cudaFree(p);
    }
};
struct Events {
    cudaEvent_t a = nullptr, b = nullptr;
    Events() { OSCB_CUDA(cudaEventCreate(&a)); OSCB_CUDA(cudaEventCreate(&b)); }
    ~Events() { if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); }
};
// exclusive scan of cnt[0..n) into out[0..n] (out[n] = total): the three passes of k_csr_scan
static void launch_scan(int64_t n, const uint32_t *cnt, int64_t *out, unsigned long long *sums, int64_t *offs, cudaStream_t s)
{
    const int64_t B = (n + 4095) / 4096;
    if (B <= 1) {
        k_csr_scan<uint32_t><<<1, 1024, 0, s>>>(n, 4096, cnt, out, nullptr, nullptr);
        return;
    }
    k_csr_scan<uint32_t><<<(unsigned)B, 1024, 0, s>>>(n, 4096, cnt, nullptr, nullptr, sums);
    k_csr_scan<unsigned long long><<<1, 1024, 0, s>>>(B, B, sums, offs, nullptr, nullptr);
    k_csr_scan<uint32_t><<<(unsigned)B, 1024, 0, s>>>(n, 4096, cnt, out, offs, nullptr);
}
} // namespace

} // namespace oscb

extern "C" int oscb_csr_from_edges(int device, int64_t n, int64_t m, const int64_t *i, const int64_t *j, const double *x,
                                   int64_t *indptr, int64_t *indices, double *data, int64_t *nnz, double *device_ms)
{
    using namespace oscb;
    try {
        OSCB_REQUIRE(n >= 1, "n must be >= 1");
        OSCB_REQUIRE(n < (int64_t)0x7fffffff && m >= 0 && m < ((int64_t)1 << 40), "graph too large for the device CSR build");
        OSCB_REQUIRE(indptr && nnz && (m == 0 || (i && j && x && indices && data)), "null buffer");
        int count = 0;
        OSCB_CUDA(cudaGetDeviceCount(&count));
        OSCB_REQUIRE(device >= 0 && device < count, "no such CUDA device: %d", device);
        OSCB_CUDA(cudaSetDevice(device));
        int sms = 0, smem_optin = 0;
        OSCB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        OSCB_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        cudaStream_t s = nullptr;                      // the legacy default stream: this call is synchronous anyway
        const size_t E = 2 * (size_t)m;

        const bool pooled = 24 * (size_t)m + 40 * E + 24 * (size_t)n <= ((size_t)512 << 20);
        Scratch<int64_t> d_i(m, pooled), d_j(m, pooled), d_indptr(n + 1, pooled), d_ocols(E, pooled);
        Scratch<double> d_x(m, pooled), d_ovals(E, pooled);
        Scratch<longlong2> d_tent(E, pooled);
        Scratch<int32_t> d_long(n, pooled);
        Scratch<uint32_t> d_deg(n, pooled), d_misc(2, pooled);         // [0] flags, [1] number of long rows
        const size_t scan_blocks = ((size_t)n + 4095) / 4096;
        Scratch<unsigned long long> d_sums(scan_blocks, pooled);
        Scratch<int64_t> d_offs(scan_blocks + 1, pooled);
        if (m) {
            OSCB_CUDA(cudaMemcpyAsync(d_i.p, i, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
            OSCB_CUDA(cudaMemcpyAsync(d_j.p, j, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
            OSCB_CUDA(cudaMemcpyAsync(d_x.p, x, m * sizeof(double), cudaMemcpyHostToDevice, s));
        }
        OSCB_CUDA(cudaMemsetAsync(d_deg.p, 0, n * sizeof(uint32_t), s));
        OSCB_CUDA(cudaMemsetAsync(d_misc.p, 0, 2 * sizeof(uint32_t), s));

        Events ev;
        float ms_a = 0.f, ms_b = 0.f;
        const int grid_e = (int)std::min<int64_t>((m + 255) / 256 + 1, (int64_t)sms * 16);
        const int grid_r = (int)std::min<int64_t>((n * 32 + 255) / 256 + 1, (int64_t)sms * 16);
        OSCB_CUDA(cudaEventRecord(ev.a, s));
        if (n <= CSR_SMEM_COUNTERS && m >= 16 * n) {
            OSCB_CUDA(cudaFuncSetAttribute(k_csr_count_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, CSR_SMEM_COUNTERS * (int)sizeof(uint32_t)));
            k_csr_count_smem<<<(int)std::min<int64_t>((m + 511) / 512, (int64_t)sms * 4), 512, (size_t)n * sizeof(uint32_t), s>>>(
                m, n, d_i.p, d_j.p, d_x.p, d_deg.p, d_misc.p);
        } else
            k_csr_count<<<grid_e, 256, 0, s>>>(m, n, d_i.p, d_j.p, d_x.p, d_deg.p, d_misc.p);
        OSCB_CUDA(cudaGetLastError());
        OSCB_CUDA(cudaEventRecord(ev.b, s));
        uint32_t misc[2] = {0, 0};
        OSCB_CUDA(cudaMemcpyAsync(misc, d_misc.p, sizeof(misc), cudaMemcpyDeviceToHost, s));
        OSCB_CUDA(cudaStreamSynchronize(s));
        OSCB_CUDA(cudaEventElapsedTime(&ms_a, ev.a, ev.b));
        // the reference's order of complaints (model.py:165-176)
        OSCB_REQUIRE(!(misc[0] & CSR_ERANGE), "coupling index out of range");
        OSCB_REQUIRE(!(misc[0] & CSR_EDIAG), "diagonal entries must be zero (no self-coupling)");
        const bool has_zero = (misc[0] & CSR_HASZERO) != 0;

        const size_t words = ((size_t)n + 31) / 32, bitmap_bytes = (words + (words + 31) / 32 + 1) * sizeof(uint32_t);
        const int bitmap_fits = bitmap_bytes <= (size_t)smem_optin ? 1 : 0;
        if (bitmap_fits)
            OSCB_CUDA(cudaFuncSetAttribute(k_csr_sort_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bitmap_bytes));
        OSCB_CUDA(cudaEventRecord(ev.a, s));
        launch_scan(n, d_deg.p, d_indptr.p, d_sums.p, d_offs.p, s);
        if (m) {
            k_csr_fill<<<grid_e, 256, 0, s>>>(m, d_i.p, d_j.p, d_x.p, d_indptr.p, d_deg.p, d_tent.p);
            // a warp per block of rows: enough warps to fill the GPU eight times over, at least 32 rows each
            const int64_t warps_wanted = std::max<int64_t>(1, std::min<int64_t>((n + 31) / 32, (int64_t)sms * 64 * 8));
            const int64_t rows_per_warp = (n + warps_wanted - 1) / warps_wanted;
            const int64_t warps = (n + rows_per_warp - 1) / rows_per_warp;
            k_csr_sort_short<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(n, rows_per_warp, d_indptr.p, d_tent.p, d_ocols.p, d_ovals.p,
                                                                        d_long.p, d_misc.p + 1, d_misc.p);
            // few long rows at a time keep many bitmaps' worth of shared memory from idling: a CTA per SM and bitmap
            const int per_sm = bitmap_fits ? std::max(1, std::min(4, (int)((size_t)smem_optin / std::max<size_t>(bitmap_bytes, 1)))) : 4;
            k_csr_sort_long<<<sms * per_sm, CSR_LONG_THREADS, bitmap_fits ? bitmap_bytes : 0, s>>>(
                n, bitmap_fits, d_indptr.p, d_tent.p, d_ocols.p, d_ovals.p, d_long.p, d_misc.p + 1, d_misc.p);
        }
        OSCB_CUDA(cudaGetLastError());
        OSCB_CUDA(cudaEventRecord(ev.b, s));
        OSCB_CUDA(cudaMemcpyAsync(misc, d_misc.p, sizeof(misc), cudaMemcpyDeviceToHost, s));
        OSCB_CUDA(cudaStreamSynchronize(s));
        OSCB_CUDA(cudaEventElapsedTime(&ms_b, ev.a, ev.b));
        OSCB_REQUIRE(!(misc[0] & CSR_EDUP), "duplicate coupling entry on an unordered pair");

        float ms_c = 0.f;
        if (!has_zero) {
            *nnz = (int64_t)E;
            OSCB_CUDA(cudaMemcpyAsync(indptr, d_indptr.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            if (E) {
                OSCB_CUDA(cudaMemcpyAsync(indices, d_ocols.p, E * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
                OSCB_CUDA(cudaMemcpyAsync(data, d_ovals.p, E * sizeof(double), cudaMemcpyDeviceToHost, s));
            }
            OSCB_CUDA(cudaStreamSynchronize(s));
        } else {
            Scratch<int64_t> d_indptr2(n + 1, pooled), d_ccols(E, pooled);
            Scratch<double> d_cvals(E, pooled);
            OSCB_CUDA(cudaEventRecord(ev.a, s));
            k_csr_nzcount<<<grid_r, 256, 0, s>>>(n, d_indptr.p, d_ovals.p, d_deg.p);
            launch_scan(n, d_deg.p, d_indptr2.p, d_sums.p, d_offs.p, s);
            k_csr_compact<<<grid_r, 256, 0, s>>>(n, d_indptr.p, d_indptr2.p, d_ocols.p, d_ovals.p, d_ccols.p, d_cvals.p);
            OSCB_CUDA(cudaGetLastError());
            OSCB_CUDA(cudaEventRecord(ev.b, s));
            OSCB_CUDA(cudaMemcpyAsync(indptr, d_indptr2.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            OSCB_CUDA(cudaStreamSynchronize(s));
            OSCB_CUDA(cudaEventElapsedTime(&ms_c, ev.a, ev.b));
            const int64_t kept = indptr[n];
            *nnz = kept;
            if (kept) {
                OSCB_CUDA(cudaMemcpyAsync(indices, d_ccols.p, kept * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
                OSCB_CUDA(cudaMemcpyAsync(data, d_cvals.p, kept * sizeof(double), cudaMemcpyDeviceToHost, s));
            }
            OSCB_CUDA(cudaStreamSynchronize(s));
        }
        if (device_ms) *device_ms = (double)ms_a + (double)ms_b + (double)ms_c;
        return OSCB_OK;
    } catch (const OscbFail &f) {
        return f.code;
    } catch (const std::exception &e) {
        set_error("oscb_csr_from_edges: %s", e.what());
        return OSCB_ECUDA;
    }
}
