// Shared helpers for the HAPOD B200 kernels (sm_100a).
//
// All matrices are float64, column-major.  An "operand" is a set of
// contiguous vectors addressed either as base + i*ld or through a device
// table of per-vector pointers (used to read a node's input as the
// concatenation of its children's mode blocks without an hstack copy,
// hierarchy.py:284-291).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>

#include "hapod_b200.h"

namespace hp {

// thread-local last error message (hp_last_error)
void set_error(const std::string& msg);
const char* last_error();

// status codes: enum hp_status of include/hapod_b200.h (HP_OK, HP_EINVAL -> ValueError,
// HP_ECUDA -> RuntimeError, HP_ELINALG -> LinAlgError, HP_ENOMEM)

#define HP_CHECK_CUDA(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::hp::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));           \
      return ::HP_ECUDA;                                                         \
    }                                                                                \
  } while (0)

// number of kernels this library launched (bench.py's gpu_launches)
void count_launches(long long n);

#define HP_CHECK_LAUNCH(what)                                                        \
  do {                                                                               \
    ::hp::count_launches(1);                                                         \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      ::hp::set_error(std::string("launch ") + (what) + ": " + cudaGetErrorString(_e)); \
      return ::HP_ECUDA;                                                         \
    }                                                                                \
  } while (0)

#define HP_REQUIRE(cond, msg)                                                        \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      ::hp::set_error(msg);                                                          \
      return ::HP_EINVAL;                                                        \
    }                                                                                \
  } while (0)

// A strided or pointer-table addressed set of vectors.
struct VecSet {
  const double* base;          // used when table == nullptr
  int64_t ld;                  // stride between vectors (elements)
  const double* const* table;  // optional device table of vector pointers
  __host__ __device__ __forceinline__ const double* vec(int64_t i) const {
    return table ? table[i] : base + i * ld;
  }
};

// ---------------------------------------------------------------- device PTX
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero fill: copies src_bytes (0..16) and zero-fills the rest.
__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------- mbarrier + TMA bulk copies
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the initialised barriers visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, int parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
// TMA bulk copy global -> shared (bytes: multiple of 16, both addresses 16-byte aligned);
// completion is signalled on `bar` as transaction bytes
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int num_sms();

// Diagnostics switched on through the C-ABI (hp_set_debug), never through the environment:
// they only add CUDA-event timing printouts and never change a result.
enum DebugFlags { DBG_JACOBI_TRACE = 1, DBG_JACOBI_ROUND_TIMING = 2, DBG_CHOL_TRACE = 4, DBG_TRI_TRACE = 8, DBG_NO_GRAPHS = 16 };
int debug_flags();

// One-time per-DEVICE setup of kernel attributes (cudaFuncSetAttribute applies to the current
// device only): each call site owns a bitmask of the devices it has configured; concurrent stream
// workers and multi-GPU processes race-free.
template <class F>
int once_per_device(std::atomic<unsigned long long>& mask, F&& setup) {
  int dev = 0;
  HP_CHECK_CUDA(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return HP_OK;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (mask.load(std::memory_order_relaxed) & bit) return HP_OK;
  const int rc = setup();
  if (rc == HP_OK) mask.fetch_or(bit, std::memory_order_release);
  return rc;
}
// Pinned host scratch of the calling host thread (allocated once, never freed per call: a
// cudaFreeHost per call would synchronise the whole device and serialise concurrent node
// streams).  512 bytes; slots: [0, 64) Jacobi sweep counters, [64, 128) re-orthonormalisation flags,
// [128, 160) pivoted Cholesky, [256, 384) tridiagonal eigensolver.
char* pinned_scratch();


// Stream-ordered zero fill as a KERNEL.  cudaMemset*Async can be serviced by a copy engine, where it
// queues behind unrelated host-to-device transfers (measured: under the e2e leg every leaf's
// 4-byte flag memset waited for most of the 13 GB upload queue); a kernel only waits for its stream.
namespace {
__global__ void zero_2d_kernel(double* p, int64_t ld, int64_t rows, int64_t cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < rows * cols) p[(e / rows) * ld + e % rows] = 0.0;
}
__global__ void zero_words_kernel(unsigned* p, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) p[e] = 0u;
}
__global__ void copy_words_kernel(unsigned* dst, const unsigned* src, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[e];
}
}  // namespace
// bytes must be a multiple of 4 (flags, counters, doubles)
inline cudaError_t zero_async(void* p, size_t bytes, cudaStream_t st) {
  const int64_t n = (int64_t)(bytes / 4);
  if (n == 0) return cudaSuccess;
  zero_words_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(static_cast<unsigned*>(p), n);
  return cudaGetLastError();
}
// Small device-to-host read into PINNED host memory (device-accessible under UVA) by a kernel:
// cudaMemcpyAsync D2H -- pinned or pageable -- was measured to queue behind the copy engine's
// pending host-to-device transfers (the e2e leaf uploads), stalling every leaf's host sync.
inline cudaError_t d2h_small(void* pinned_dst, const void* src, size_t bytes, cudaStream_t st) {
  const int64_t n = (int64_t)(bytes / 4);
  if (n == 0) return cudaSuccess;
  copy_words_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(static_cast<unsigned*>(pinned_dst),
                                                                 static_cast<const unsigned*>(src), n);
  return cudaGetLastError();
}
inline cudaError_t zero_2d_async(double* p, int64_t ld, int64_t rows, int64_t cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  zero_2d_kernel<<<(unsigned)ceil_div(rows * cols, 256), 256, 0, st>>>(p, ld, rows, cols);
  return cudaGetLastError();
}

}  // namespace hp
