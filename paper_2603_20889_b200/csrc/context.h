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
  double* xbuf = nullptr;  // resident copy of X for the *_host entry points
  size_t xbuf_doubles = 0;
  double* gen = nullptr;  // scratch of sqb_generate_dev
  size_t gen_doubles = 0;

  sqb::StatusWord* d_status = nullptr;
  sqb::StatusWord* h_status = nullptr;  // pinned mirror
  long long last_index = -1;
  long long launches = 0;

  // NCCL (resolved with dlopen on first use; single-GPU paths never touch it)
  void* nccl_comm = nullptr;
  bool own_comm = false;
  int rank = 0;
  int world = 1;
};
