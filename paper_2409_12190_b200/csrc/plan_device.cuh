// The symbolic phase on the device (plan_device.cu): the plan of plan.cpp
// (+ the tile classes and index blobs of problem.cu) for a single-rank
// problem, built from the observation arrays already in device memory.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>

#include "device.cuh"

namespace bae {

struct DevicePlan {
  // host scalars
  int T = 0, E = 0, n_small = 0, n_big = 0, blob_bytes = 0;
  int max_tile_obs = 0, max_tile_cams = 0, max_tile_pts = 0;
  int big_need = 0;                  // largest workspace of a big tile (bytes)
  int kind_slice[kWsKindCount] = {};  // largest small-tile workspace per kernel kind (bytes)
  bool has_empty_camera = false, has_empty_point = false;
  // device arrays (from the caller's allocator), as Dev / Plan
  int *tile_obs_begin = nullptr, *tile_pt_begin = nullptr, *tile_ent_begin = nullptr, *tile_ws = nullptr;
  std::uint32_t* obs_lcpt = nullptr;
  int* obs_orig = nullptr;
  int *ent_cam = nullptr, *ent_obs_begin = nullptr, *cam_ent_ptr = nullptr, *cam_ent = nullptr;
  int* pt_ptr = nullptr;
  std::uint16_t* ptobs = nullptr;
  int* pt_of_internal = nullptr;
  int4* tile_desc = nullptr;
  char* tile_blob = nullptr;
  int *small_tiles = nullptr, *big_tiles = nullptr;
};

// cam / pt: the N observation indices in device memory. Throws
// Error(BAE_ERR_INDEX, position) for the lowest observation with an index out
// of range, as validate_inputs does. slice_limit: the largest per-warp
// workspace of a small tile (problem.cu kSliceLimit). Synchronises s.
void build_plan_device(int C, int P, const int* cam, const int* pt, long long N, int tile_obs_cap, int tile_cam_cap,
                       int tile_pts_cap, long long slice_limit, const std::function<void*(std::size_t)>& alloc,
                       cudaStream_t s, DevicePlan& out);

}  // namespace bae
