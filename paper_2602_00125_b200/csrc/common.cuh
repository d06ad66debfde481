// Shared plumbing for libb2: error capture, streams, launch accounting.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <string>

#include "../../include/b2.h"

namespace b2 {

void set_error(const std::string& msg);
int fail(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
cudaStream_t resolve(void* stream);
int sm_count();
constexpr int kTickets = 4096;
constexpr int kGemmTicket = kTickets;           // GEMM unit scheduler: [draw counter, done counter]
constexpr int kTicketsAlloc = kTickets + 64;
unsigned* tickets(cudaStream_t st);  // zeroed per-stream arrival counters (kTicketsAlloc)
int ensure_init();
// SMs the persistent GEMM grids use: all of them, minus the ones reserved
// (b2_gemm_set_sm_reserve) for kernels that must run beside the GEMMs --
// NCCL's collectives during a data-parallel backward.
int gemm_sms();

// One tensor-core GEMM problem (gemm_tc.cu); up to 3 run in one launch.
struct TcDesc {
  int ta, tb;
  int64_t M, N, K;
  const void *a0, *a1, *a2;
  int64_t lda;
  const void *b0, *b1, *b2;
  int64_t ldb;
  float* C;
  int64_t ldc;
  const float* bias;
  int epi;
  const float* mask;
  void* s_hi;
  void* s_lo;
  float* colsum;
  const uint64_t* mask_bits;
  uint64_t* bits_out;
};
int gemm_tc_group(int mode, const TcDesc* d, int n, cudaStream_t st);
extern std::atomic<uint64_t> g_launches;

inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// check a launch, count it, map errors to a status
inline int launched(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, what);
  count_launch();
  return 0;
}

// grid sizing: a multiple of the SM count (148 on B200) x resident CTAs
inline int grid_for(int64_t work_items, int per_cta, int ctas_per_sm = 4) {
  int64_t need = (work_items + per_cta - 1) / per_cta;
  int64_t cap = (int64_t)sm_count() * ctas_per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

}  // namespace b2

#define B2_TRY(expr)                      \
  do {                                    \
    int _rc = (expr);                     \
    if (_rc != 0) return _rc;             \
  } while (0)

#define B2_CUDA(expr)                                  \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return b2::cuda_fail(_e, #expr); \
  } while (0)

// Collapsed N-d iteration descriptor (dims merged where strides allow).
struct B2Shape {
  int ndim;
  int64_t shape[B2_MAX_DIMS];
  int64_t st[3][B2_MAX_DIMS];  // up to 3 operands (out + 2 inputs)
};
