// Tile-sparse Cholesky of the reduced camera system S (the direct solver,
// SolverChoice::cholesky, lm.hpp:132-136; the reference factors the full
// system with an AMD-ordered sparse Cholesky, cholesky.hpp:77-281).
//
// S (6C x 6C, camera order) is cut into kTB x kTB tiles (8 cameras per tile;
// the last tile is padded with an identity). Only the tiles of L's fill
// pattern are stored (column-major inside a tile). The pattern comes from a
// tile-level symbolic factorisation done once per problem (plan_tile_chol).
//
// Numeric factorisation is ONE persistent kernel, left-looking by tile
// column: CTAs claim columns in ascending (topological) order from an atomic
// work counter, so a column that waits for its subtree never holds back
// columns that are ready (list scheduling; every lower column is already
// claimed, hence no deadlock). Column j first finishes its diagonal tile (the updates from every
// column k with L(j,k) != 0, waiting on the epoch flag of that tile), factors
// and inverts it and performs its step of the forward substitution L y = b;
// then each tile below the diagonal gets its updates, is solved against
// L(j,j)^-T and published with its own flag, so the next column starts as
// soon as the one tile it needs exists. There is no grid-wide barrier:
// independent parts of the elimination tree run concurrently. A second
// dataflow kernel runs the backward substitution L^T x = y in descending
// column order. Every sum runs in a fixed order: results are bitwise
// reproducible.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace bae {

constexpr int kTB = 48;              // tile edge (8 cameras)
constexpr int kTT = kTB * kTB;       // doubles per tile
// Failure word values: 1 = a pivot was not positive (NotSpdError); kCholTimeout
// = a flag wait exceeded kFlagTimeoutNs (a lost producer; BAE_ERR_CUDA).
constexpr int kCholTimeout = 2;
constexpr unsigned long long kFlagTimeoutNs = 20ull * 1000 * 1000 * 1000;
constexpr int kCholThreads = 256;    // 16 x 16 threads, 3 x 3 outputs each

// Host-side symbolic structure (plan_tile_chol).
struct TileCholPlan {
  int nt = 0;                       // tile columns
  int n = 0;                        // true order (6C); rows >= n are padding
  std::vector<int> colptr;          // nt+1: L tiles of column j, diagonal first, rows ascending
  std::vector<int> rowidx;          // tile row of each stored tile (slot = position)
  std::vector<int> rptr;            // nt+1: row structure of column j: k < j with L(j,k) != 0
  std::vector<int> rk, rslot;       // k in (level(k), k) order, slot of L(j,k)
  std::vector<int> level;           // per column: 1 + the highest level of its k (0: no updates)
  std::vector<int> uptr;            // per row-structure entry q: range of its tile updates
  std::vector<int> usrc, udst;      // update: C(udst) -= L(usrc) L(rslot[q])^T
  // per column, all its updates ordered by (k, target tile):
  // {target position in the column (0 = diagonal), source slot L(i,k), slot of L(j,k), q}
  std::vector<int> bptr;            // nt+1
  std::vector<int> bop;             // 4 per update
  long long nnz_tiles() const { return static_cast<long long>(rowidx.size()); }
};

// Fill-reducing order of the camera graph (cameras joined when they see a
// common point): nested dissection by BFS level sets -- a pseudo-peripheral
// start, the middle level as separator, the two sides recursively, the
// separator last. Groups are returned in elimination order; every group is
// later padded to whole tiles, so independent subtrees never share a tile
// and the elimination tree's height drops from O(C) to O(log C) separator
// levels for banded / sequential camera graphs. Small or dense subgraphs
// stay one group (BFS order).
std::vector<std::vector<int>> nd_camera_groups(int C, const std::vector<std::pair<int, int>>& edges, int leaf);

// Update helpers: a tile below the diagonal whose column holds at least
// `min_ops` updates into it from columns other than the column's last
// contributing one (k_last) gets a helper task -- another CTA applies those
// updates (same order, same arithmetic: bitwise the same tile) while the
// column's owner works on its diagonal, so a separator column's dozens of
// tile updates no longer run on one SM. Tasks are {column, target position
// (0: the owner), first op, end op}, in queue order (a column's helpers just
// before its owner; every task only waits on tasks queued before it). `bptr`
// / `bop` are rewritten: the owner's ops per column, then the helpers' ops.
struct TileCholTasks {
  std::vector<int> tasks;            // 4 per task
  std::vector<unsigned> hmask;       // per column: bit s set when tile position s has a helper
  std::vector<int> bptr, bop;        // the owner's ops per column, then the helper ranges
  std::vector<int> order;            // the columns in queue order (the backward takes it reversed)
  int helpers = 0;
};
// Only the queue's last `tail_tasks` tasks (the grid size) get helpers.
TileCholTasks plan_chol_tasks(const TileCholPlan& pl, int min_ops, int tail_tasks);

// Tile-level symbolic Cholesky from the lower-triangular tile pattern of S:
// `lower_pairs` lists tile pairs (i, j), i >= j (duplicates allowed); every
// diagonal tile is included automatically.
TileCholPlan plan_tile_chol(int n, const std::vector<std::pair<int, int>>& lower_pairs);

// Device view.
struct TileChol {
  int nt, n;            // n = 6 * positions (padded, tile-aligned groups)
  int nnz;              // stored tiles
  const int* colptr;
  const int* rowidx;
  const int* rptr;
  const int* rk;
  const int* rslot;
  const int* uptr;
  const int* usrc;
  const int* udst;
  const int* bptr;
  const int* bop;
  double* tiles;        // nnz_tiles * kTT; diagonal slots receive L(j,j)^-1 after the factorisation
  const double* rhs;    // right-hand side, camera order (6 per camera)
  double* y;            // nt * kTB forward-substitution result
  double* x;            // solution, camera order (6 per camera)
  const int* pos_cam;   // camera at each position (n / 6), -1 for a padding slot
  const unsigned long long* padmask;  // per tile: bit r set when row r is padding (unit pivot)
  unsigned* flags;      // nnz + nt epoch flags: one per stored tile (factor), one per column (backward)
  unsigned* pflags;     // nnz: a helper's tile is pre-updated (or null without helpers)
  const int* tasks;     // 4 per task (plan_chol_tasks), or null: task i = column i, no helpers
  const unsigned* hmask;  // per column helper positions (with tasks)
  const int* border;    // backward: column of the s-th claim (the queue's columns reversed), or null
  int ntask;
  unsigned* next;       // 3 words: work counters (factor, backward; CTAs claim columns in topological
                        // order) and the epoch, the flag value of the current solve
  int* fail;            // 1: a pivot is not positive (NotSpdError, cholesky.hpp:229); kCholTimeout
  unsigned long long* trace;  // BAE_CHOL_TRACE: 8 globaltimer stamps per column, or null
};

// Factor + solve on stream s (three launches: counters and epoch, factor,
// backward); the epoch lives on the device (next[2]), so the sequence can be
// captured in a graph and replayed.
int launch_tile_chol(const TileChol& t, int grid, cudaStream_t s);
int tile_chol_grid(int ntask);

}  // namespace bae
