// Device construction of the direct solver's pair list (pairs.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "device.cuh"

namespace bae {

// Keeps the device's default memory pool from returning its memory at every
// synchronisation (the pair list's stream-ordered scratch).
void pairs_pool_setup();

// Per internal point the number of its (k, l) pairs with c(k) >= c(l),
// exclusive-scanned into off[0..P]; returns the total (synchronises s).
// With `blocks` (C * C bits, zeroed), also marks every camera block (c1, c2),
// c1 >= c2, that has a pair.
long long count_pairs(const Dev& d, long long* off, cudaStream_t s, unsigned* blocks = nullptr);

// The marked camera blocks in (c1, c2) order -- the block list build_pairs
// returns, known before the pair sort (synchronises s).
std::vector<int2> marked_blocks(const Dev& d, const unsigned* blocks, cudaStream_t s);

// The pairs grouped by camera block (c1, c2) ascending, generation order
// inside a block, into pairs[0..np); the blocks' cameras and pair offsets to
// the host (synchronises s).
void build_pairs(const Dev& d, const long long* off, long long np, int2* pairs, std::vector<int2>& bcam,
                 std::vector<int>& bptr, cudaStream_t s);

}  // namespace bae
