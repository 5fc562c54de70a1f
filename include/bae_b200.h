/*
 * bae_b200.h -- C ABI of the B200-native bundle-adjustment hot path.
 *
 * This is the drop-in boundary for the reference library's BA/LM entry points
 * (traceopt, /root/reference/proj/include/traceopt). The reference is a
 * header-only C++ API with no FFI of its own; each entry point below names the
 * reference function it replaces. Plain pointers and sizes only; no C++ or
 * torch types cross this boundary and no exceptions escape it: the reference
 * exception classes (errors.hpp:10-69) map to the BAE_ERR_* return codes, and
 * the offending position/observation is available from bae_last_error_index().
 *
 * Threading: a handle is used from one host thread at a time (the reference
 * runs one orchestrating caller thread). Independent handles
 * may be used concurrently.
 *
 * Layouts (all host buffers, row-major, FP64 unless noted):
 *   pose   : 7 doubles [tx, ty, tz, qx, qy, qz, qw], world->camera
 *            (trace.hpp:318-326 write_pose). Quaternions are taken as-is
 *            (read_pose uses QuatRotation::from_unit, trace.hpp:329-333).
 *   point  : 3 doubles [x, y, z]
 *   intr   : 3 doubles [f, k1, k2] (BalIntrinsics, camera.hpp:23-25), or with
 *            camera_model = BAE_CAMERA_PINHOLE 4 doubles [fx, fy, cx, cy]
 *            (PinholeIntrinsics, camera.hpp:17-19)
 *   pixel  : 2 doubles per observation
 *   indices: int32 camera / point index per observation (problems.hpp:19-23)
 */
#ifndef BAE_B200_H_
#define BAE_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes (errors.hpp:10-69 + device-side failures). */
#define BAE_OK 0
#define BAE_ERR_INVALID_ARGUMENT 1    /* std::invalid_argument                    */
#define BAE_ERR_INDEX 2               /* IndexError(position)  problems.hpp:105-110 */
#define BAE_ERR_CHEIRALITY 3          /* CheiralityError(observation) camera.hpp:51 */
#define BAE_ERR_NOT_SPD 4             /* NotSpdError(pivot)                        */
#define BAE_ERR_NUMERICAL_BREAKDOWN 5 /* NumericalBreakdownError                   */
#define BAE_ERR_UNSUPPORTED 6         /* UnsupportedOperationError                 */
#define BAE_ERR_CUDA 7                /* CUDA runtime failure (no device, OOM ...) */
#define BAE_ERR_NCCL 8                /* NCCL failure                              */
#define BAE_ERR_PARSE 9               /* ParseError(line)       errors.hpp:60-69    */
#define BAE_ERR_IO 10                 /* a file cannot be opened / written         */

/* LmConfig::solver (lm.hpp:20). */
#define BAE_SOLVER_CHOLESKY 0
#define BAE_SOLVER_PCG 1

/* CameraIntrinsics variant of a problem (camera.hpp:17-27; one per problem, problems.hpp:94-98). */
#define BAE_CAMERA_BAL 0
#define BAE_CAMERA_PINHOLE 1

/* TerminationReason (lm.hpp:21). */
#define BAE_TERM_PLATEAU 0
#define BAE_TERM_MAX_ITERS 1
#define BAE_TERM_SOLVER_FAILURE 2

/* = LmConfig (lm.hpp:23-38); defaults from bae_lm_config_default(). */
typedef struct bae_lm_config {
  double initial_damping; /* 1e-6  */
  double damping_min;     /* 1e-16 */
  double damping_max;     /* 1e16  */
  double damping_up;      /* 2.0   */
  double damping_down;    /* 0.5   */
  double clamp_min;       /* 1e-6  */
  double clamp_max;       /* 1e32  */
  double plateau_rel_tol; /* 1e-6  */
  double pcg_tol;         /* 1e-8  relative to the full rhs -J^T r (pcg.hpp:85) */
  int64_t pcg_max_iters;  /* 0: max(250, 2 * (cameras + points)), lm.hpp:139-142 */
  int32_t max_iterations; /* 10    */
  int32_t plateau_patience; /* 3   */
  int32_t solver;         /* BAE_SOLVER_*; the reference default is cholesky  */
  int32_t use_caches;     /* 1 (symbolic reuse; the GPU path always caches)   */
} bae_lm_config;

/* ⊇ LmIterationRecord (lm.hpp:62-69); entry 0 is the initial state. */
typedef struct bae_iter_record {
  int32_t iteration;
  int32_t accepted;
  double cost;       /* accepted-history cost after this iteration */
  double mse;        /* cost / residual rows (lm.hpp:214)          */
  double lambda;     /* damping used by this iteration's solve     */
  double cum_time_s; /* wall seconds since the loop started        */
  int64_t pcg_iters; /* inner iterations of this step (extension)  */
  double grad_norm;  /* ||J^T r|| at the linearisation point (ext) */
  double trial_cost; /* cost of the tentative step (inf = rejected by cheirality) */
} bae_iter_record;

/* = LmReport (lm.hpp:71-77) minus the trajectory vector. */
typedef struct bae_lm_report {
  double final_cost;
  double final_mse;
  int32_t iterations;
  int32_t reason; /* BAE_TERM_* */
  int32_t accepted_steps;
  int32_t rejected_steps;
  double final_lambda;
  double solve_seconds;   /* wall time of the LM loop (lm.hpp:222-232) */
  int64_t total_pcg_iters;
  double device_seconds;  /* CUDA-event time of the LM loop on the solver stream */
} bae_lm_report;

/* Creation options (no reference counterpart; NULL = defaults). */
typedef struct bae_create_options {
  int32_t device;      /* CUDA ordinal, default 0                                  */
  int32_t tile_obs;    /* observations per tile (0 = auto)                        */
  int32_t jacobian;    /* 0 = recompute blocks in every pass, 1 = store J in HBM  */
  int32_t rank;        /* distributed: this rank (default 0)                      */
  int32_t world;       /* distributed: number of ranks (default 1)                */
  int32_t camera_model; /* BAE_CAMERA_BAL (default; intrinsics C x [f, k1, k2]) or
                           BAE_CAMERA_PINHOLE (C x [fx, fy, cx, cy]); camera.hpp:17-27 */
  const void* nccl_id; /* distributed: 128-byte ncclUniqueId from rank 0 (one process per GPU) */
  struct bae_group* group; /* distributed: in-process rank group (one host thread per rank) */
} bae_create_options;

typedef struct bae_problem bae_problem;
typedef struct bae_group bae_group;

/* ---- library -------------------------------------------------------------- */
const char* bae_version(void);
void bae_lm_config_default(bae_lm_config* cfg);
void bae_create_options_default(bae_create_options* opt);
/* Message / index of the last failure on this host thread (any entry point). */
const char* bae_last_error(void);
int64_t bae_last_error_index(void);
/* ---- landmark-sharded problems ------------------------------
 * A problem created with world > 1 (or with an NCCL id / rank group) is
 * sharded by landmark: every rank passes the WHOLE problem to bae_create_ba
 * and keeps the points bae_partition_points assigns to it, with all their
 * observations; cameras are replicated. Per LM iteration the ranks sum the
 * camera blocks (27 C + 2 doubles) and, per PCG iteration, the reduced-system
 * product (6 C doubles); every rank then holds identical camera-side state and
 * takes identical decisions, so each entry point below must be called by all
 * ranks together (collective calls), with the same arguments' nullness.
 * Exports that are per observation (residual vector, Jacobian, transpose
 * plans, block diagonals, bae_solve_step) return BAE_ERR_UNSUPPORTED.
 * Backends: NCCL (one process per GPU; rank 0 calls bae_nccl_unique_id and
 * broadcasts the 128 bytes with its own launcher) or an in-process rank group
 * (one host thread per rank, on one or several peer-enabled GPUs). */
/* 128-byte NCCL unique id for bae_create_options.nccl_id (rank 0 creates it;
 * NCCL is loaded at run time, BAE_ERR_NCCL if libnccl.so.2 is absent). */
int bae_nccl_unique_id(void* out128);
/* In-process rank group of `world` ranks (1..16) for bae_create_options.group.
 * Reference counted: the caller's handle and every problem created with it
 * own it, so bae_group_destroy may come before the problems are destroyed. */
int bae_group_create(int32_t world, bae_group** out);
void bae_group_destroy(bae_group* g);

/* ---- pose graph (make_pgo_problem, problems.hpp:141-188) -- */
/* Edges (i, j, measurement T as a pose7) with the residual
 * Log(z_i^-1 z_j T^-1) (trace.hpp:475-487); information36 (nullable) holds a
 * row-major 6x6 information matrix per edge, used where has_information[k]
 * != 0 (NULL = every edge): residual rows are whitened by L^T of its Cholesky
 * factor (problems.hpp:169-184). anchor_first holds pose 0 fixed. The
 * handle works with bae_optimize (poses only; points NULL; solver =
 * cholesky), bae_evaluate (6 residuals per edge), bae_set/get_parameters,
 * bae_num_poses, bae_residual_rows (= edges). */
int bae_create_pgo(const double* poses7, int32_t num_poses, const int32_t* edge_i, const int32_t* edge_j,
                   const double* measurements7, const double* information36, const int32_t* has_information,
                   int64_t num_edges, int32_t anchor_first, const bae_create_options* opts, bae_problem** out);
/* Per edge d r_w / d pose_i and d r_w / d pose_j (row-major 6x6 each; the
 * reverse pass of trace.hpp:657-671), for parity tests. */
int bae_pgo_jacobian(bae_problem* p, double* jacobian_i36, double* jacobian_j36);

/* ---- problem (make_ba_problem, problems.hpp:87-136) ------------------------- */
/* Validates like the reference (intrinsics count, empty observations,
 * IndexError with the observation position, camera index checked first) and
 * evaluates the initial residual, so a point on the camera plane fails here
 * with BAE_ERR_CHEIRALITY and the lowest offending observation, exactly as the
 * reference's eager forward at graph construction does (trace.hpp:464-474). */
int bae_create_ba(const double* poses7, int32_t num_cameras, const double* points3,
                  int32_t num_points, const double* bal_intrinsics3, const int32_t* cam_idx,
                  const int32_t* pt_idx, const double* pixels2, int64_t num_observations,
                  const bae_create_options* opts, bae_problem** out);
void bae_destroy(bae_problem* p);

int32_t bae_num_poses(const bae_problem* p);    /* TracedProblem::num_poses   */
int32_t bae_num_points(const bae_problem* p);   /* TracedProblem::num_points  */
int64_t bae_residual_rows(const bae_problem* p);/* TracedProblem::residual_rows */

/* TracedProblem::set_parameters (problems.hpp:61-64). */
int bae_set_parameters(bae_problem* p, const double* poses7, const double* points3);
int bae_get_parameters(bae_problem* p, double* poses7, double* points3);
/* TracedProblem::evaluate (problems.hpp:66) + squared_norm (lm.hpp:81-85).
 * residuals2 (nullable) receives r = projection - pixel in observation order. */
int bae_evaluate(bae_problem* p, double* residuals2, double* cost);
/* TracedProblem::jacobian (problems.hpp:68, trace.hpp:553-806): the two BSR
 * halves of JacobianPair. The pattern is read back from the device's
 * observation decomposition: row_ptr counts the block rows the device holds
 * per observation (0..N when each row is one block, as trace.hpp:728-790
 * builds it); col arrays are the gather indices. Any output pointer may be
 * NULL. */
int bae_jacobian(bae_problem* p, double* jpose_2x6, double* jpoint_2x3,
                 int64_t* pose_row_ptr, int32_t* pose_col, int64_t* point_row_ptr,
                 int32_t* point_col);
/* transpose_symbolic (bsr.hpp:140-160) of one Jacobian half, which = 0 pose /
 * 1 point: row_ptr (num_cols+1), col_idx (N, observation ids ascending within
 * each row), src_block (N). This is the camera / point segmentation the
 * device reductions use. */
int bae_transpose_plan(bae_problem* p, int32_t which, int64_t* row_ptr, int32_t* col_idx,
                       int64_t* src_block);
/* Block pattern of one quadrant of A = J^T J, which = 0 CC, 1 CL, 2 LC, 3 LL
 * (spgemm_symbolic, spgemm.hpp:33-81, as NormalEquations::initialize builds
 * them, assemble.hpp:47-53), or with which = 4 the scalar CSR pattern of A
 * (build_csr_pattern, assemble.hpp:135-177). The device never forms CL / LC
 * (implicit Schur); the patterns are derived from its observation
 * decomposition, read back from device memory. rows / nnz are always written;
 * row_ptr (rows+1) and col_idx (nnz) when non-NULL. Single-rank problems. */
int bae_normal_pattern(bae_problem* p, int32_t which, int64_t* rows, int64_t* nnz, int64_t* row_ptr,
                       int32_t* col_idx);
/* Damped normal-equation pieces for parity (assemble.hpp:61-101): per-camera
 * 6x6 H_cc and 6-vector g_c = J_c^T r, per-point 3x3 H_pp and g_p, undamped,
 * at the current parameters. Any output may be NULL. */
int bae_block_diagonals(bae_problem* p, double* hcc36, double* gc6, double* hpp9, double* gp3);

/* ---- optimizer (optimize, lm.hpp:205-255) ----------------------------------- */
/* traj receives min(iterations+1, traj_cap) records; poses_out / points_out
 * (nullable) receive the optimised parameters, which the handle also keeps
 * (lm.hpp:250-252). */
int bae_optimize(bae_problem* p, const double* init_poses7, const double* init_points3,
                 const bae_lm_config* cfg, bae_iter_record* traj, int32_t traj_cap,
                 bae_lm_report* report, double* poses_out, double* points_out);

/* ---- one damped solve (lm.hpp:126-145) --------------------------------------- */
/* Linearises at the current parameters, damps with lambda and solves with
 * cfg->solver: the tile-sparse Cholesky of the reduced camera system
 * (BAE_SOLVER_CHOLESKY, the reference default) or the implicit-Schur PCG
 * (BAE_SOLVER_PCG); delta receives [6C pose tangents | 3P point deltas] in
 * the reference's column order (lm.hpp:159-173). */
int bae_solve_step(bae_problem* p, double lambda, const bae_lm_config* cfg, double* delta,
                   int64_t* pcg_iters, double* rel_residual);

/* ---- plateau rule, exposed for host-logic tests (lm.hpp:89-108) -------------- */
int bae_stop_on_plateau(const double* history, int64_t n, const bae_lm_config* cfg,
                        int32_t* stop);

/* ---- synthetic BAL-shaped scene (io/synthetic.hpp conventions) - */
/* Deterministic from the seed. Writes the parsed BAL-equivalent problem:
 * initial poses7 / points3 / intrinsics3 / observations (camera-major), and the
 * ground truth (true_poses7, true_points3; nullable). num_observations must be
 * >= 2 * num_points and <= num_points * min(num_cameras, 16). */
int bae_synth_bal_shaped(int32_t num_cameras, int32_t num_points, int64_t num_observations,
                         uint64_t seed, double pixel_sigma, double pose_sigma,
                         double point_sigma, double* poses7, double* points3,
                         double* intrinsics3, int32_t* cam_idx, int32_t* pt_idx,
                         double* pixels2, double* true_poses7, double* true_points3);
/* The same scene family generated on the device (row f4): every value from
 * Philox4x32-10 keyed by the seed, counter = (stream, entity, draw), one
 * thread per point / camera / observation (csrc/synth_device.cu documents the
 * streams). Not the host generator's values (that one follows the reference
 * Rng stream); the oracle restates this one for the tests. */
int bae_synth_bal_shaped_device(int32_t num_cameras, int32_t num_points, int64_t num_observations,
                                uint64_t seed, double pixel_sigma, double pose_sigma, double point_sigma,
                                int32_t device, double* poses7, double* points3, double* intrinsics3,
                                int32_t* cam_idx, int32_t* pt_idx, double* pixels2, double* true_poses7,
                                double* true_points3);

/* ---- BAL files, the reference's synthetic scene, the CLI - */
typedef struct bae_bal bae_bal;
/* parse_bal (io/bal.hpp:103-142) of a file / a text buffer (a file may also
 * be the binary cache of bae_bal_write_binary). ParseError ->
 * BAE_ERR_PARSE with bae_last_error_index() = line (the reference's messages
 * and line numbers); an unopenable file -> BAE_ERR_IO. */
int bae_bal_read(const char* path, bae_bal** out);
int bae_bal_parse(const char* text, int64_t len, bae_bal** out);
/* synth_ba (io/synthetic.hpp:46-91): every camera sees every point. */
int bae_bal_synthetic(int32_t num_cameras, int32_t num_points, double pixel_noise, double pose_noise,
                      uint64_t seed, bae_bal** out);
/* A BalProblem from arrays; cameras9 = C x [rodrigues3, translation3, f, k1, k2]. */
int bae_bal_from_arrays(int32_t num_cameras, int32_t num_points, int64_t num_observations, const double* cameras9,
                        const double* points3, const int32_t* cam_idx, const int32_t* pt_idx, const double* pixels2,
                        bae_bal** out);
int bae_bal_counts(const bae_bal* b, int32_t* num_cameras, int32_t* num_points, int64_t* num_observations);
/* Arrays of the problem (any may be NULL): poses7 / intrinsics3 through
 * BalCamera::pose / intrinsics (io/bal.hpp:24-27), points, observations, and
 * the raw 9-scalar camera records. */
int bae_bal_arrays(const bae_bal* b, double* poses7, double* intrinsics3, double* points3, int32_t* cam_idx,
                   int32_t* pt_idx, double* pixels2, double* cameras9);
/* serialize_bal (io/bal.hpp:145-157): %.17g, round-trips doubles exactly. */
int bae_bal_write(const bae_bal* b, const char* path);
/* Binary problem cache (no reference counterpart): the
 * parsed arrays with a magic header. bae_bal_read (and so the CLI's --input)
 * recognises the format and loads it without the text scanner. */
int bae_bal_write_binary(const bae_bal* b, const char* path);
void bae_bal_free(bae_bal* b);
/* parse_g2o (io/g2o.hpp:30-80): VERTEX_SE3:QUAT / EDGE_SE3:QUAT, edge
 * endpoints remapped to vertex positions, identity information elided
 * (has_information = 0), unknown tags kept as warnings; ParseError ->
 * BAE_ERR_PARSE with the line. */
typedef struct bae_g2o bae_g2o;
int bae_g2o_read(const char* path, bae_g2o** out);
int bae_g2o_parse(const char* text, int64_t len, bae_g2o** out);
int bae_g2o_counts(const bae_g2o* g, int32_t* num_vertices, int64_t* num_edges, int32_t* num_warnings);
int bae_g2o_arrays(const bae_g2o* g, double* poses7, int64_t* vertex_ids, int32_t* edge_i, int32_t* edge_j,
                   double* measurements7, double* information36, int32_t* has_information);
const char* bae_g2o_warning(const bae_g2o* g, int32_t k);
void bae_g2o_free(bae_g2o* g);
/* write_csv (cli.hpp:69-79): iter,cost,mse,lambda,accepted,cum_time_s. */
int bae_write_csv(const char* path, const bae_iter_record* traj, int32_t n);
/* cli_main (cli.hpp:116-200): `ba` / `pgo` subcommands, the reference's flags
 * (+ --device), summary line and exit codes (0 ok, 1 usage, 2 data error,
 * 3 solver failure). paper_2409_12190_b200/traceopt_bench wraps it. */
int bae_cli_main(int argc, const char* const* argv);

/* ---- direct-solver host logic, exposed for tests ---------------------------- */
/* Nested-dissection order of a camera graph (edges2 = pairs of cameras):
 * order (C) lists the cameras group by group in elimination order,
 * group_ptr (C + 1) the group boundaries. */
int bae_nd_order(int32_t num_cameras, int64_t num_edges, const int32_t* edges2, int32_t leaf, int32_t* order,
                 int32_t* group_ptr, int32_t* num_groups);
/* Tile-level symbolic Cholesky of an nt x nt tile pattern (pairs2 = lower
 * tile pairs (i, j), i >= j): colptr (nt + 1) and rowidx (nnz, diagonal first,
 * rows ascending) of L's tiles. */
int bae_tile_symbolic(int32_t nt, int64_t num_pairs, const int32_t* pairs2, int32_t* colptr, int32_t* rowidx,
                      int64_t capacity, int64_t* nnz);
/* Work queue of the tile factorisation with update helpers (host logic of
 * plan_chol_tasks, for tests): the original per-column update lists
 * (orig_bptr nt + 1, orig_ops 4 per update: target position, L(i,k) slot,
 * L(j,k) slot, row-structure entry), the rewritten lists (bptr: the owner's
 * updates per column; ops: owners first, then the helper ranges), the tasks
 * (4 each: column, helper position or 0 for the owner, first op, end op) and
 * the per-column helper masks. capacity bounds ops, orig_ops and tasks. */
int bae_chol_tasks(int32_t nt, int64_t num_pairs, const int32_t* pairs2, int32_t min_ops, int32_t tail_tasks,
                   int64_t capacity, int32_t* orig_bptr, int32_t* orig_ops, int32_t* bptr, int32_t* ops,
                   int32_t* tasks, int32_t* num_tasks, uint32_t* hmask);

/* ---- multi-GPU landmark partition, host only ----------------- */
/* Contiguous ranges of the internal point order balanced by observation
 * count: rank_of_point[p] in [0, world). Cameras are replicated. */
int bae_partition_points(int32_t num_cameras, int32_t num_points, const int32_t* cam_idx, const int32_t* pt_idx,
                         int64_t num_observations, int32_t world, int32_t* rank_of_point);

/* ---- measurement hooks (bench.py) ------------------------------------------ */
/* Device-timed (CUDA events on the solver stream) averages over `reps`
 * launches: kind 0 = linearisation (fused residual + Jacobian + block
 * reductions), 1 = one implicit Schur S*x product (one PCG iteration's
 * operator), 2 = one full PCG iteration, 3 = fused residual+Jacobian to HBM
 * (stored J), 4 = tile-sparse Cholesky factorisation + forward/backward
 * substitution of the reduced camera system (direct solver), 5 = the direct
 * solver's prep (damped point blocks, V = W L^-T, right-hand side), 6 = its
 * Schur assembly, 7 = kinds 0 and 5 fused into one pass (what an LM
 * iteration after an accepted step runs; single rank), 8 = the trial (camera
 * retraction, point back-substitution, trial cost). ms receives the mean
 * milliseconds per launch. */
int bae_time_kernel(bae_problem* p, int32_t kind, int32_t reps, double* ms);
/* Number of kernel launches issued by this handle since creation. */
int64_t bae_launch_count(const bae_problem* p);
/* Device milliseconds accumulated per LM phase since the last reset:
 * [linearize, prep, assemble (direct), factor+solve (direct), pcg, trial,
 * commit]; reset != 0 clears after reading. */
int bae_phase_times(bae_problem* p, double* ms7, int32_t reset);
/* This handle's shard: rank, world, points and observations it owns. */
int bae_problem_shard(const bae_problem* p, int32_t* rank, int32_t* world, int32_t* local_points,
                      int64_t* local_observations);
/* The plan's device arrays (single rank), for parity of the device and the
 * host planner: which = 0 tile_obs_begin, 1 tile_pt_begin, 2 tile_ent_begin,
 * 3 tile_ws, 4 obs_lcpt, 5 obs_orig, 6 ent_cam, 7 ent_obs_begin,
 * 8 cam_ent_ptr, 9 cam_ent, 10 pt_ptr, 11 ptobs (2-byte), 12 pt_of_internal,
 * 13 tile_desc (4 ints per tile), 14 small_tiles, 15 big_tiles, 16 pixels in
 * slot order (doubles), 17 launch shapes (slice, warps per CTA per kernel
 * kind, big tiles, big stride, empty camera, empty point, max tile
 * observations), 18 index blobs (bytes). *count = elements, *elem_bytes =
 * their size; out (capacity cap elements) may be NULL. */
int bae_plan_array(bae_problem* p, int32_t which, void* out, int64_t cap, int64_t* count, int32_t* elem_bytes);
/* Direct solver structure (after its first use): [tile columns, stored
 * 48x48 tiles, tile updates, nested-dissection groups, camera positions]. */
int bae_direct_stats(const bae_problem* p, int64_t* out5);
/* Schur assembly size (after the direct solver's first use): the (k, l)
 * observation pairs and the 6x6 camera blocks they sum into. */
int bae_direct_pairs(const bae_problem* p, int64_t* pairs, int64_t* blocks);
/* Static sizes the roofline arithmetic needs: [N, P, C, tiles, tile-camera
 * entries, max obs per tile]. */
int bae_problem_stats(const bae_problem* p, int64_t* out6);

#ifdef __cplusplus
}
#endif

#endif /* BAE_B200_H_ */
