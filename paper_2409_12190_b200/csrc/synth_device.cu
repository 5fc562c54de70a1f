// On-device BAL-shaped scenes. The host generator
// (synth.cpp) draws from one sequential Mersenne-twister stream -- the
// reference Rng, so its scenes match the oracle's -- which takes seconds at
// Final-13682 size. This generator keeps the same scene (unit-box points, a
// radius-4 ring of inward-looking cameras, f = 500, k1 ~ U(-0.1, 0.1),
// k2 ~ U(-0.01, 0.01), banded visibility by a partial Fisher-Yates shuffle of
// a window of min(C, 16) cameras, exactly N observations ordered camera-major,
// exact projections + pixel noise, poses retracted by tangent noise, points
// moved by point noise) but draws every value from Philox4x32-10 keyed by the
// seed with the counter (stream, entity, draw), so each point, camera and
// observation is one thread and the scene does not depend on the launch
// shape. Streams (draw n gives two 64-bit words a, b):
//   1 point p:   n=0 (x, y), n=1 (z)            true point -0.5 + u01
//   2 camera c:  n=0 Box-Muller(a, b) -> height 0.5 + 0.1 g; n=1 k1, k2
//   3 point j:   n=0 anchor a % C; draw i of the shuffle: n = 1 + i/2, word a (i even) / b (i odd)
//   4 obs k:     n=0 Box-Muller pair -> pixel noise (u, v)   (k in the final camera-major order)
//   5 camera c:  n=0..2 Box-Muller pairs -> tangent noise tau[0..5]
//   6 point p:   n=0 pair -> (x, y), n=1 cos branch -> z       point noise
// Box-Muller: g = sqrt(-2 ln(1 - u01(a))) (cos | sin)(2 pi u01(b)).
// The oracle restates the same algorithm on the host (oracle/bae_oracle.cpp,
// or_synth_bal_shaped_philox); tests/test_gpu_synth.py compares them.
#include <cub/device/device_radix_sort.cuh>

#include <climits>
#include <string>
#include <vector>

#include "bae/philox.hpp"
#include "bae_internal.hpp"
#include "lie.cuh"

namespace bae {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(BAE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// products and sums rounded separately (no FMA contraction), as on the host
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ void box_muller(const PhiloxWords& w, double& g0, double& g1) {
  const double r = sqrt(mul(-2.0, log(1.0 - philox_u01(w.a))));
  const double th = mul(2.0 * M_PI, philox_u01(w.b));
  g0 = mul(r, cos(th));
  g1 = mul(r, sin(th));
}

// look_at_origin (io/synthetic.hpp:26-38) as synth.cpp states it, device side.
__device__ bool look_at(const P3& pos, Q4& q, P3& t) {
  const double n = sqrt(add(add(mul(pos.x, pos.x), mul(pos.y, pos.y)), mul(pos.z, pos.z)));
  const P3 zc{pos.x / n, pos.y / n, pos.z / n};
  P3 up{0, 0, 1};
  if (fabs(add(add(mul(up.x, zc.x), mul(up.y, zc.y)), mul(up.z, zc.z))) > 0.95) up = {0, 1, 0};
  P3 xc{add(mul(up.y, zc.z), -mul(up.z, zc.y)), add(mul(up.z, zc.x), -mul(up.x, zc.z)),
        add(mul(up.x, zc.y), -mul(up.y, zc.x))};
  const double xn = sqrt(add(add(mul(xc.x, xc.x), mul(xc.y, xc.y)), mul(xc.z, xc.z)));
  xc = {xc.x / xn, xc.y / xn, xc.z / xn};
  const P3 yc{add(mul(zc.y, xc.z), -mul(zc.z, xc.y)), add(mul(zc.z, xc.x), -mul(zc.x, xc.z)),
              add(mul(zc.x, xc.y), -mul(zc.y, xc.x))};
  const double m[9] = {xc.x, xc.y, xc.z, yc.x, yc.y, yc.z, zc.x, zc.y, zc.z};
  double c[4];
  double tr = add(add(m[0], m[4]), m[8]);
  if (tr > 0.0) {
    tr = sqrt(add(tr, 1.0));
    c[3] = mul(0.5, tr);
    tr = 0.5 / tr;
    c[0] = mul(add(m[7], -m[5]), tr);
    c[1] = mul(add(m[2], -m[6]), tr);
    c[2] = mul(add(m[3], -m[1]), tr);
  } else {
    int i = 0;
    if (m[4] > m[0]) i = 1;
    if (m[8] > m[i * 4]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    tr = sqrt(add(add(add(m[i * 4], -m[j * 4]), -m[k * 4]), 1.0));
    c[i] = mul(0.5, tr);
    tr = 0.5 / tr;
    c[3] = mul(add(m[k * 3 + j], -m[j * 3 + k]), tr);
    c[j] = mul(add(m[j * 3 + i], m[i * 3 + j]), tr);
    c[k] = mul(add(m[k * 3 + i], m[i * 3 + k]), tr);
  }
  if (!quat_normalize(c[0], c[1], c[2], c[3], q)) return false;
  t = {-add(add(mul(m[0], pos.x), mul(m[1], pos.y)), mul(m[2], pos.z)),
       -add(add(mul(m[3], pos.x), mul(m[4], pos.y)), mul(m[5], pos.z)),
       -add(add(mul(m[6], pos.x), mul(m[7], pos.y)), mul(m[8], pos.z))};
  return true;
}

struct SynDev {
  int C, P, W;
  long long N, base, extra;
  unsigned long long seed;
  double pix_sigma, pose_sigma, pt_sigma;
  double *tpts, *pts, *tq, *tt, *poses, *tposes, *intr, *px;
  int *vis_cam, *vis_pt, *cam_idx, *pt_idx;
  int* bad;  // lowest failing entity (camera plane / degenerate camera)
};

__global__ void k_syn_points(SynDev s) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= s.P) return;
  const PhiloxWords w0 = philox_words(s.seed, 1, p, 0), w1 = philox_words(s.seed, 1, p, 1);
  const double x = add(-0.5, philox_u01(w0.a)), y = add(-0.5, philox_u01(w0.b)), z = add(-0.5, philox_u01(w1.a));
  double g0, g1, g2, unused;
  box_muller(philox_words(s.seed, 6, p, 0), g0, g1);
  box_muller(philox_words(s.seed, 6, p, 1), g2, unused);
  s.tpts[3LL * p] = x;
  s.tpts[3LL * p + 1] = y;
  s.tpts[3LL * p + 2] = z;
  s.pts[3LL * p] = add(x, mul(s.pt_sigma, g0));
  s.pts[3LL * p + 1] = add(y, mul(s.pt_sigma, g1));
  s.pts[3LL * p + 2] = add(z, mul(s.pt_sigma, g2));
}

__global__ void k_syn_cams(SynDev s) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= s.C) return;
  double h, unused;
  box_muller(philox_words(s.seed, 2, c, 0), h, unused);
  const PhiloxWords wk = philox_words(s.seed, 2, c, 1);
  const double ang = mul(2.0 * M_PI, static_cast<double>(c)) / s.C;
  const P3 pos{mul(4.0, cos(ang)), mul(4.0, sin(ang)), add(0.5, mul(0.1, h))};
  Q4 q;
  P3 t;
  if (!look_at(pos, q, t)) {
    atomicMin(s.bad, c);
    return;
  }
  s.intr[3LL * c] = 500.0;
  s.intr[3LL * c + 1] = add(-0.1, mul(0.2, philox_u01(wk.a)));
  s.intr[3LL * c + 2] = add(-0.01, mul(0.02, philox_u01(wk.b)));
  double tau[6];
  for (int d = 0; d < 3; ++d) {
    double g0, g1;
    box_muller(philox_words(s.seed, 5, c, d), g0, g1);
    tau[2 * d] = mul(s.pose_sigma, g0);
    tau[2 * d + 1] = mul(s.pose_sigma, g1);
  }
  Q4 q1;
  P3 t1;
  if (!se3_retract(q, t, tau, q1, t1)) {
    atomicMin(s.bad, c);
    return;
  }
  // BAL camera record: Rodrigues vector, then BalCamera::pose's se3_exp
  const P3 rod = so3_log(q1);
  const double tau_rot[6] = {0, 0, 0, rod.x, rod.y, rod.z};
  Q4 qb;
  P3 unused3;
  se3_exp(tau_rot, qb, unused3);
  double* o = s.poses + 7LL * c;
  o[0] = t1.x;
  o[1] = t1.y;
  o[2] = t1.z;
  o[3] = qb.x;
  o[4] = qb.y;
  o[5] = qb.z;
  o[6] = qb.w;
  double* g = s.tposes + 7LL * c;
  g[0] = t.x;
  g[1] = t.y;
  g[2] = t.z;
  g[3] = q.x;
  g[4] = q.y;
  g[5] = q.z;
  g[6] = q.w;
  s.tq[4LL * c] = q.x;
  s.tq[4LL * c + 1] = q.y;
  s.tq[4LL * c + 2] = q.z;
  s.tq[4LL * c + 3] = q.w;
  s.tt[3LL * c] = t.x;
  s.tt[3LL * c + 1] = t.y;
  s.tt[3LL * c + 2] = t.z;
}

// Point j's cameras, point-major at j base + min(j, extra).
__global__ void k_syn_vis(SynDev s) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s.P) return;
  const int m = static_cast<int>(s.base + (j < s.extra ? 1 : 0));
  const long long at = static_cast<long long>(j) * s.base + min(static_cast<long long>(j), s.extra);
  const int a = static_cast<int>(philox_words(s.seed, 3, j, 0).a % static_cast<unsigned long long>(s.C));
  int window[16];
  for (int i = 0; i < s.W; ++i) window[i] = (a + i) % s.C;
  PhiloxWords w{0, 0};
  for (int i = 0; i < m; ++i) {
    if ((i & 1) == 0) w = philox_words(s.seed, 3, j, 1 + i / 2);
    const unsigned long long word = (i & 1) ? w.b : w.a;
    const int r = i + static_cast<int>(word % static_cast<unsigned long long>(s.W - i));
    const int tmp = window[i];
    window[i] = window[r];
    window[r] = tmp;
    s.vis_cam[at + i] = window[i];
    s.vis_pt[at + i] = j;
  }
}

__global__ void k_syn_pixels(SynDev s) {
  const long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (k >= s.N) return;
  const int c = s.cam_idx[k], p = s.pt_idx[k];
  const Q4 q{s.tq[4LL * c], s.tq[4LL * c + 1], s.tq[4LL * c + 2], s.tq[4LL * c + 3]};
  const P3 y = quat_rotate(q, P3{s.tpts[3LL * p], s.tpts[3LL * p + 1], s.tpts[3LL * p + 2]});
  double u = 0, v = 0;
  if (!bal_project(P3{add(y.x, s.tt[3LL * c]), add(y.y, s.tt[3LL * c + 1]), add(y.z, s.tt[3LL * c + 2])},
                   s.intr[3LL * c], s.intr[3LL * c + 1], s.intr[3LL * c + 2], u, v)) {
    atomicMin(s.bad, static_cast<int>(k));
    return;
  }
  double g0, g1;
  box_muller(philox_words(s.seed, 4, k, 0), g0, g1);
  s.px[2 * k] = add(u, mul(s.pix_sigma, g0));
  s.px[2 * k + 1] = add(v, mul(s.pix_sigma, g1));
}

}  // namespace

void synth_bal_shaped_device(int C, int P, std::int64_t N, std::uint64_t seed, double pixel_sigma, double pose_sigma,
                             double point_sigma, int device, double* poses7, double* points3, double* intr3,
                             std::int32_t* cam_idx, std::int32_t* pt_idx, double* px2, double* true_poses7,
                             double* true_points3) {
  if (C < 1 || P < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "synth: counts must be positive");
  const int W = std::min(C, 16);
  if (N < 2 * std::int64_t{P} && C >= 2)
    throw Error(BAE_ERR_INVALID_ARGUMENT, "synth: need at least two observations per point");
  if (N > std::int64_t{P} * W) throw Error(BAE_ERR_INVALID_ARGUMENT, "synth: too many observations for window");
  if (N >= (std::int64_t{1} << 31) - 1) throw Error(BAE_ERR_UNSUPPORTED, "synth: more than 2^31-2 observations");
  ck(cudaSetDevice(device), "cudaSetDevice");
  cudaStream_t st;
  ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  SynDev s{};
  s.C = C;
  s.P = P;
  s.W = W;
  s.N = N;
  s.base = N / P;
  s.extra = N % P;
  s.seed = seed;
  s.pix_sigma = pixel_sigma;
  s.pose_sigma = pose_sigma;
  s.pt_sigma = point_sigma;
  std::vector<void*> bufs;
  auto dal = [&](std::size_t bytes) {
    void* p = nullptr;
    ck(cudaMallocAsync(&p, std::max<std::size_t>(bytes, 16), st), "cudaMallocAsync");
    bufs.push_back(p);
    return p;
  };
  try {
    const std::size_t Cs = C, Ps = P, Ns = static_cast<std::size_t>(N);
    s.tpts = static_cast<double*>(dal(24 * Ps));
    s.pts = static_cast<double*>(dal(24 * Ps));
    s.tq = static_cast<double*>(dal(32 * Cs));
    s.tt = static_cast<double*>(dal(24 * Cs));
    s.poses = static_cast<double*>(dal(56 * Cs));
    s.tposes = static_cast<double*>(dal(56 * Cs));
    s.intr = static_cast<double*>(dal(24 * Cs));
    s.px = static_cast<double*>(dal(16 * Ns));
    s.vis_cam = static_cast<int*>(dal(4 * Ns));
    s.vis_pt = static_cast<int*>(dal(4 * Ns));
    s.cam_idx = static_cast<int*>(dal(4 * Ns));
    s.pt_idx = static_cast<int*>(dal(4 * Ns));
    s.bad = static_cast<int*>(dal(sizeof(int)));
    const int big = INT_MAX;
    ck(cudaMemcpyAsync(s.bad, &big, sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    k_syn_points<<<(P + 255) / 256, 256, 0, st>>>(s);
    k_syn_cams<<<(C + 127) / 128, 128, 0, st>>>(s);
    k_syn_vis<<<(P + 255) / 256, 256, 0, st>>>(s);
    ck(cudaGetLastError(), "synth kernels");
    int bits = 1;
    while (bits < 31 && (C >> bits) != 0) ++bits;
    std::size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, s.vis_cam, s.cam_idx, s.vis_pt, s.pt_idx, N, 0, bits, st);
    void* tmp = dal(tb);
    // stable by camera: points stay ascending inside a camera (camera-major, like BAL files)
    ck(cub::DeviceRadixSort::SortPairs(tmp, tb, s.vis_cam, s.cam_idx, s.vis_pt, s.pt_idx, N, 0, bits, st),
       "camera-major sort");
    k_syn_pixels<<<static_cast<unsigned>((N + 255) / 256), 256, 0, st>>>(s);
    ck(cudaGetLastError(), "synth pixels");
    int bad = INT_MAX;
    ck(cudaMemcpyAsync(&bad, s.bad, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "synth");
    if (bad != INT_MAX) throw Error(BAE_ERR_CHEIRALITY, "synth: point on camera plane", bad);
    auto down = [&](void* dst, const void* src, std::size_t bytes) {
      if (dst) ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "D2H scene");
    };
    down(poses7, s.poses, 56 * Cs);
    down(points3, s.pts, 24 * Ps);
    down(intr3, s.intr, 24 * Cs);
    down(cam_idx, s.cam_idx, 4 * Ns);
    down(pt_idx, s.pt_idx, 4 * Ns);
    down(px2, s.px, 16 * Ns);
    down(true_poses7, s.tposes, 56 * Cs);
    down(true_points3, s.tpts, 24 * Ps);
    ck(cudaStreamSynchronize(st), "synth D2H");
  } catch (...) {
    for (void* p : bufs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    throw;
  }
  for (void* p : bufs) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
}

}  // namespace bae
