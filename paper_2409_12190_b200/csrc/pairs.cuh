// Device construction of the direct solver's pair list (pairs.cu).
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <vector>

#include "device.cuh"

namespace bae {

// Keeps the device's default memory pool from returning its memory at every
// synchronisation (the pair list's stream-ordered scratch).
void pairs_pool_setup();

// Per internal point the number of its (k, l) pairs with c(k) >= c(l),
// exclusive-scanned into off[0..P]; returns the total (synchronises s).
long long count_pairs(const Dev& d, long long* off, cudaStream_t s);

// The pairs grouped by camera block (c1, c2) ascending, generation order
// inside a block, into pairs[0..np); the blocks' cameras and pair offsets to
// the host (synchronises s).
void build_pairs(const Dev& d, const long long* off, long long np, int2* pairs, std::vector<int2>& bcam,
                 std::vector<int>& bptr, cudaStream_t s);

}  // namespace bae

namespace bae {

struct Plan;

// Supertiles of the Schur assembly (k_schur_super) and their units, host side.
struct SuperHost {
  std::vector<int4> sup_a, sup_b;
  std::vector<int2> sup_chunk, unit_pr;
  std::vector<int> blk_uptr, blk_units;
  std::vector<int2> chunk_meta;          // per chunk {supertile or -1 (single), first unit slot}
  std::vector<int> cta_chunk, cta_nreg;  // persistent CTA ranges (whole supertiles) and their regular chunks
  int regular = 0, single = 0;
  long long units = 0;
  // device (from the caller's allocator): the staged chunks' pair blobs
  // and per chunk {blob byte offset / 16, blob bytes}
  char* blob = nullptr;
  int2* chunk_blob = nullptr;
  long long blob_bytes = 0;
};

// Cuts the plan's warp-tiles into supertiles, re-sorts the block-grouped pair
// list (device, `pairs`, block b at [bptr[b], bptr[b+1])) into (supertile,
// block, point) order as supertile-local k | l << 16 words into spairs[0..np),
// and forms the units (synchronises s).
void build_super(const Dev& d, const Plan& pl, const int2* pairs, const int* blk_ptr_dev, const std::vector<int>& bptr,
                 long long np, unsigned* spairs, SuperHost& out, int grid,
                 const std::function<void*(std::size_t)>& alloc, cudaStream_t s);

}  // namespace bae
