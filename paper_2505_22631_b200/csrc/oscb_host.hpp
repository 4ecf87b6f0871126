// oscb_host.hpp -- host-side plumbing shared by the translation units of liboscb.so:
// error reporting, RAII device buffers and the graph handle behind `oscb_graph`.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdarg.h>
#include <stdio.h>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/oscb.h"

namespace oscb {

void set_error(const char *fmt, ...);

struct OscbFail {
    int code;
};

#define OSCB_CUDA(expr)                                                                        \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            ::oscb::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
            throw ::oscb::OscbFail{e_ == cudaErrorMemoryAllocation ? OSCB_ENOMEM : OSCB_ECUDA}; \
        }                                                                                      \
    } while (0)

#define OSCB_REQUIRE(cond, ...)                                                                \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            ::oscb::set_error(__VA_ARGS__);                                                    \
            throw ::oscb::OscbFail{OSCB_EINVAL};                                               \
        }                                                                                      \
    } while (0)

// Size-keyed pool of device blocks: oscb_run allocates a dozen workspaces per call and
// cudaMalloc / cudaFree cost about a millisecond each (and synchronise the device), which is as
// much as a whole short integrate window.  Freed blocks are parked per (device, bytes) and handed
// back to the next request of the same size; oscb_pool_trim() really frees them.
void *pool_alloc(size_t bytes);
void pool_free(void *p, size_t bytes);
void pool_trim();

// device buffer that returns its block to the pool; sized in elements of T
template <typename T> struct DevBuf {
    T *p = nullptr;
    size_t count = 0;
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), count(o.count) { o.p = nullptr; o.count = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept
    {
        if (this != &o) { release(); p = o.p; count = o.count; o.p = nullptr; o.count = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void release()
    {
        if (p) pool_free(p, count * sizeof(T));
        p = nullptr;
        count = 0;
    }
    void alloc(size_t n)
    {
        release();
        if (n == 0) n = 1;
        p = static_cast<T *>(pool_alloc(n * sizeof(T)));
        count = n;
    }
    void upload(const T *src, size_t n, cudaStream_t s)
    {
        if (n) OSCB_CUDA(cudaMemcpyAsync(p, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void download(T *dst, size_t n, cudaStream_t s) const
    {
        if (n) OSCB_CUDA(cudaMemcpyAsync(dst, p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    void zero(cudaStream_t s) { OSCB_CUDA(cudaMemsetAsync(p, 0, count * sizeof(T), s)); }
};

struct ResidentPlan; // oscb_resident_host.hpp
struct DensePlan;    // oscb_dense_host.hpp
struct ShardWork;    // oscb.cu: workspace of the row-sharded dense driver
struct UmmaPlan;     // oscb_umma.hpp: tile images of J for the tensor-core dense kernel
struct LowdegPlan;   // oscb_lowdeg_host.hpp: slot map + ELL stream of the low-degree kernel

// numpy's Philox4x64 initial phases of replicas `seeds` into phi [R][n] float64 (k_initial_phases, oscb.cu)
void launch_initial_phases(const uint64_t *d_seeds, double *d_phi, int n, int R, cudaStream_t s);

} // namespace oscb

// The handle behind the opaque `oscb_graph`.
struct oscb_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sm_count = 0;
    int smem_optin = 0; // max dynamic shared memory per block (opt-in), bytes
    int64_t n = 0, nnz = 0, pairs = 0, max_degree = 0;
    int64_t row_begin = 0, row_end = 0;
    bool is_dense = false, unit_weights = false, int_weights = false;

    // host mirror of the canonical CSR (int32 indices) -- used to build kernel-specific plans
    std::vector<int> h_indptr, h_indices;
    std::vector<double> h_w;

    // device CSR + canonical pairs (model.py:238-242)
    oscb::DevBuf<int> d_indptr, d_indices, d_iu, d_jv;
    oscb::DevBuf<double> d_w64, d_pw;
    oscb::DevBuf<float> d_w32;
    oscb::DevBuf<unsigned long long> d_nonfinite;

    // resident-kernel plans keyed by (precision, replicas_per_cta, threads)
    std::map<uint64_t, std::shared_ptr<oscb::ResidentPlan>> plans;
    std::map<uint64_t, std::shared_ptr<oscb::LowdegPlan>> lowdeg_plans;
    std::shared_ptr<oscb::DensePlan> dense;
    std::shared_ptr<oscb::ShardWork> shard_work;
    std::shared_ptr<oscb::UmmaPlan> umma;
};
