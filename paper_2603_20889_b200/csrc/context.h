// Context object behind the C ABI (include/skinnyqr_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

struct sqb_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  cudaStream_t own_stream_handle = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D slab copies of the *_host entry points
  cudaEvent_t slab_ready = nullptr;
  int sm_count = 0;

  // growable device workspaces
  double* work = nullptr;  // stacked triangles Y / per-CTA partial Grams (two halves, ping-pong)
  size_t work_doubles = 0;
  double* small = nullptr;  // n x n scratch matrices for the drivers
  size_t small_doubles = 0;
  double* xbuf = nullptr;  // resident copy of X: two-pass *_host entry points (CholQR2, SVQB2, ...)
  size_t xbuf_doubles = 0;
  // single-pass *_host entry points stream X through a ring of row slabs instead (O(slab) state)
  static constexpr int kRing = 3;
  double* ring = nullptr;
  size_t ring_doubles = 0;
  cudaEvent_t ring_free[kRing] = {nullptr, nullptr, nullptr};
  long long host_slab_bytes = 256ll << 20;  // slab size of the host-pointer paths (sqb_set_host_slab_bytes)
  double* qslab = nullptr;  // row slab of Q = X F for the 129..256-column fused sweeps
  size_t qslab_doubles = 0;
  double* gen = nullptr;  // scratch of sqb_generate_dev
  size_t gen_doubles = 0;

  sqb::StatusWord* d_status = nullptr;
  sqb::StatusWord* h_status = nullptr;  // pinned mirror
  long long last_index = -1;
  long long launches = 0;

  int tsqr_kind = -1;  // forced TSQR kernel family (sqb_set_tsqr_kernel), -1 = selection table

  // Row-sharded runs: the n x n exchange goes through NCCL (resolved with dlopen on first use;
  // single-GPU paths never touch it) or through a caller-supplied all-gather (sqb_set_allgather).
  void* nccl_comm = nullptr;
  bool own_comm = false;
  int rank = 0;
  int world = 1;
  sqb_allgather_fn gather_fn = nullptr;
  void* gather_user = nullptr;
};
