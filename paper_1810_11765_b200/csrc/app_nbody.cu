// app_nbody.cu -- N-body with collisions (Table 1, Listing 1 P:143-183;
// reading R-NBODY).  Type 0 = Body{x, y, vx, vy, fx, fy, m: f32; id, target,
// incoming: u32; merged: u8} (41 B, N_T = 64).
//
// device_do -- the sequential all-bodies loop inside each
// body's method -- becomes a tiled all-pairs gather over an id-indexed SOA
// snapshot S (x, y, m, vx, vy, handle) that a preceding do-all writes: each
// CTA stages 256 snapshot entries in shared memory and every thread sums its
// body's interactions tile by tile in id order (same terms as the paper's
// loop, deterministic order).  Dead ids have m = 0 in S and contribute 0.
#include "dsr_host.h"

namespace dsr {

enum { NB_X = 0, NB_Y, NB_VX, NB_VY, NB_FX, NB_FY, NB_M, NB_ID, NB_TARGET, NB_INCOMING, NB_MERGED };
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kTile = 256;

template <class V>
__device__ __forceinline__ V& bf(const DevHeap& h, uint32_t b, uint32_t s, int f) {
  return *field_ptr<V>(h, 0, (uint32_t)f, b, s);
}

// ---- parallel_new<Body>(n): body i gets id id_offset + i
__global__ void __launch_bounds__(256) k_nb_new(DevHeap h, uint64_t n, dsr_nbody_args a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t nh = dsr_new(h, 0);
    if (!nh) continue;
    const uint32_t b = h_bid(nh), s = h_slot(nh);
    bf<float>(h, b, s, NB_X) = a.x0[i];
    bf<float>(h, b, s, NB_Y) = a.y0[i];
    bf<float>(h, b, s, NB_VX) = a.vx0[i];
    bf<float>(h, b, s, NB_VY) = a.vy0[i];
    bf<float>(h, b, s, NB_FX) = 0.f;
    bf<float>(h, b, s, NB_FY) = 0.f;
    bf<float>(h, b, s, NB_M) = a.m0[i];
    bf<uint32_t>(h, b, s, NB_ID) = a.id_offset + (uint32_t)i;
    bf<uint32_t>(h, b, s, NB_TARGET) = kNone;
    bf<uint32_t>(h, b, s, NB_INCOMING) = kNone;
    bf<uint8_t>(h, b, s, NB_MERGED) = 0;
  }
}

__global__ void k_nb_clear(uint64_t n, dsr_nbody_args a) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    a.sm[i] = 0.f;
    a.shandle[i] = 0;
  }
}

struct NbSnapshot {
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t id = bf<uint32_t>(h, b, s, NB_ID);
    a.sx[id] = bf<float>(h, b, s, NB_X);
    a.sy[id] = bf<float>(h, b, s, NB_Y);
    a.sm[id] = bf<float>(h, b, s, NB_M);
    a.svx[id] = bf<float>(h, b, s, NB_VX);
    a.svy[id] = bf<float>(h, b, s, NB_VY);
    a.shandle[id] = make_handle(0, h.types[0].cap, b, s);
  }
};

// compute_force: f_i = G m_i sum_j m_j (p_j - p_i) / (|p_j - p_i|^2 + eps^2)^{3/2}
__global__ void __launch_bounds__(kTile) k_nb_force(DevHeap h, dsr_nbody_args a) {
  __shared__ float4 tile[kTile];
  const uint32_t n = a.n;
  const float eps2 = a.eps * a.eps;
  for (uint32_t base = blockIdx.x * kTile; base < n; base += gridDim.x * kTile) {
    const uint32_t i = base + threadIdx.x;
    float xi = 0.f, yi = 0.f;
    uint64_t hi = 0;
    if (i < n) { hi = a.shandle[i]; xi = a.sx[i]; yi = a.sy[i]; }
    float ax = 0.f, ay = 0.f;
    for (uint32_t j0 = 0; j0 < n; j0 += kTile) {
      __syncthreads();
      const uint32_t j = j0 + threadIdx.x;
      tile[threadIdx.x] = j < n ? make_float4(a.sx[j], a.sy[j], a.sm[j], 0.f) : make_float4(0.f, 0.f, 0.f, 0.f);
      __syncthreads();
      const uint32_t lim = (n - j0) < (uint32_t)kTile ? (n - j0) : (uint32_t)kTile;
#pragma unroll 8
      for (uint32_t k = 0; k < lim; ++k) {
        const float4 p = tile[k];
        const float dx = p.x - xi, dy = p.y - yi;
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, eps2));
        const float inv = rsqrtf(r2);
        const float w = p.z * inv * inv * inv;
        ax = fmaf(dx, w, ax);
        ay = fmaf(dy, w, ay);
      }
    }
    if (hi) {
      const uint32_t b = h_bid(hi), s = h_slot(hi);
      const float gm = a.G * bf<float>(h, b, s, NB_M);
      bf<float>(h, b, s, NB_FX) = gm * ax;
      bf<float>(h, b, s, NB_FY) = gm * ay;
    }
  }
}

struct NbMove {   // semi-implicit Euler, velocity first
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const float m = bf<float>(h, b, s, NB_M);
    const float vx = bf<float>(h, b, s, NB_VX) + bf<float>(h, b, s, NB_FX) / m * a.dt;
    const float vy = bf<float>(h, b, s, NB_VY) + bf<float>(h, b, s, NB_FY) / m * a.dt;
    bf<float>(h, b, s, NB_VX) = vx;
    bf<float>(h, b, s, NB_VY) = vy;
    bf<float>(h, b, s, NB_X) = bf<float>(h, b, s, NB_X) + vx * a.dt;
    bf<float>(h, b, s, NB_Y) = bf<float>(h, b, s, NB_Y) + vy * a.dt;
    bf<uint32_t>(h, b, s, NB_TARGET) = kNone;
    bf<uint32_t>(h, b, s, NB_INCOMING) = kNone;
    bf<uint8_t>(h, b, s, NB_MERGED) = 0;
  }
};

// prepare_merge: target_i = argmin_{j : (m_j, j) >lex (m_i, i), d2 < R^2} (d2, j)
__global__ void __launch_bounds__(kTile) k_nb_merge_search(DevHeap h, dsr_nbody_args a) {
  __shared__ float4 tile[kTile];
  const uint32_t n = a.n;
  const float R2 = a.R * a.R;
  for (uint32_t base = blockIdx.x * kTile; base < n; base += gridDim.x * kTile) {
    const uint32_t i = base + threadIdx.x;
    float xi = 0.f, yi = 0.f, mi = 0.f;
    uint64_t hi = 0;
    if (i < n) { hi = a.shandle[i]; xi = a.sx[i]; yi = a.sy[i]; mi = a.sm[i]; }
    uint32_t best = kNone;
    float bestd = 0.f;
    for (uint32_t j0 = 0; j0 < n; j0 += kTile) {
      __syncthreads();
      const uint32_t j = j0 + threadIdx.x;
      tile[threadIdx.x] = j < n ? make_float4(a.sx[j], a.sy[j], a.sm[j], 0.f) : make_float4(0.f, 0.f, 0.f, 0.f);
      __syncthreads();
      if (!hi) continue;
      const uint32_t lim = (n - j0) < (uint32_t)kTile ? (n - j0) : (uint32_t)kTile;
      for (uint32_t k = 0; k < lim; ++k) {
        const float4 p = tile[k];
        const float dx = p.x - xi, dy = p.y - yi;
        const float d2 = fmaf(dx, dx, dy * dy);
        const uint32_t jj = j0 + k;
        const bool heavier = p.z > mi || (p.z == mi && jj > i);
        if (heavier && p.z > 0.f && d2 < R2 && (best == kNone || d2 < bestd)) { best = jj; bestd = d2; }
      }
    }
    if (hi) bf<uint32_t>(h, h_bid(hi), h_slot(hi), NB_TARGET) = best;
  }
}

struct NbClaim {  // at most one absorption per target per step: smallest id wins
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t t = bf<uint32_t>(h, b, s, NB_TARGET);
    if (t == kNone) return;
    const uint64_t ht = a.shandle[t];
    atomicMin(&bf<uint32_t>(h, h_bid(ht), h_slot(ht), NB_INCOMING), bf<uint32_t>(h, b, s, NB_ID));
  }
};

struct NbAbsorb { // perfectly inelastic merge: momentum and centre of mass
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t i = bf<uint32_t>(h, b, s, NB_INCOMING);
    if (i == kNone || bf<uint32_t>(h, b, s, NB_TARGET) != kNone) return;
    const float m = bf<float>(h, b, s, NB_M), mi = a.sm[i];
    const float mn = m + mi;
    bf<float>(h, b, s, NB_VX) = (m * bf<float>(h, b, s, NB_VX) + mi * a.svx[i]) / mn;
    bf<float>(h, b, s, NB_VY) = (m * bf<float>(h, b, s, NB_VY) + mi * a.svy[i]) / mn;
    bf<float>(h, b, s, NB_X) = (m * bf<float>(h, b, s, NB_X) + mi * a.sx[i]) / mn;
    bf<float>(h, b, s, NB_Y) = (m * bf<float>(h, b, s, NB_Y) + mi * a.sy[i]) / mn;
    bf<float>(h, b, s, NB_M) = mn;
    const uint64_t hi = a.shandle[i];
    bf<uint8_t>(h, h_bid(hi), h_slot(hi), NB_MERGED) = 1;
  }
};

struct NbDeleteMerged {   // step_6_delete_merged
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args&, Acc&) {
    if (bf<uint8_t>(h, b, s, NB_MERGED)) dsr_destroy(h, make_handle(0, h.types[0].cap, b, s));
  }
};

struct NbDump {
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    float* o = a.out + 6ull * bf<uint32_t>(h, b, s, NB_ID);
    o[0] = bf<float>(h, b, s, NB_X);
    o[1] = bf<float>(h, b, s, NB_Y);
    o[2] = bf<float>(h, b, s, NB_VX);
    o[3] = bf<float>(h, b, s, NB_VY);
    o[4] = bf<float>(h, b, s, NB_M);
    o[5] = 1.f;
  }
};

bool nb_method_info(uint32_t id, MethodInfo* mi) {
  if (id >= DSR_M_NB_SNAPSHOT && id <= DSR_M_NB_DUMP) { *mi = {0, sizeof(dsr_nbody_args)}; return true; }
  return false;
}

bool nb_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args) {
  const dsr_nbody_args& a = *(const dsr_nbody_args*)args;
  switch (id) {
    case DSR_M_NB_SNAPSHOT: launch_doall<NbSnapshot>(c, T, snapshot, args); return true;
    case DSR_M_NB_FORCE: {
      const int g = (int)((a.n + kTile - 1) / kTile);
      k_nb_force<<<g < c.sms * 8 ? g : c.sms * 8, kTile, 0, c.st>>>(c.h, a);
      count_launch();
      return true;
    }
    case DSR_M_NB_MOVE: launch_doall<NbMove>(c, T, snapshot, args); return true;
    case DSR_M_NB_PREPARE_MERGE: {
      const int g = (int)((a.n + kTile - 1) / kTile);
      k_nb_merge_search<<<g < c.sms * 8 ? g : c.sms * 8, kTile, 0, c.st>>>(c.h, a);
      count_launch();
      return true;
    }
    case DSR_M_NB_CLAIM: launch_doall<NbClaim>(c, T, snapshot, args); return true;
    case DSR_M_NB_ABSORB: launch_doall<NbAbsorb>(c, T, snapshot, args); return true;
    case DSR_M_NB_DELETE_MERGED: launch_doall<NbDeleteMerged>(c, T, snapshot, args); return true;
    case DSR_M_NB_DUMP: launch_doall<NbDump>(c, T, snapshot, args); return true;
  }
  return false;
}

bool nb_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok) {
  *ok = 1;
  if (id != DSR_K_NB_CLEAR_SNAPSHOT) return false;
  if (bytes != sizeof(dsr_nbody_args)) { *ok = 0; return true; }
  k_nb_clear<<<grid_for(c, n), 256, 0, c.st>>>(n, *(const dsr_nbody_args*)args);
  count_launch();
  return true;
}

bool nb_ctor_launch(uint32_t id, const LaunchCtx& c, uint32_t T, uint64_t n, const void* args, size_t bytes, int* ok) {
  *ok = 1;
  if (id != DSR_C_NB_BODY) return false;
  if (bytes != sizeof(dsr_nbody_args) || T != 0) { *ok = 0; return true; }
  k_nb_new<<<grid_for(c, n), 256, 0, c.st>>>(c.h, n, *(const dsr_nbody_args*)args);
  count_launch();
  return true;
}

}  // namespace dsr
