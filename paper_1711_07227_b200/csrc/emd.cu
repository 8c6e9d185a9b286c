// Exact word mover's distance for batches of document pairs (emd.py:120-211):
// the balanced transportation problem solved by successive shortest augmenting
// paths with node potentials -- multi-source Dijkstra over reduced costs clamped
// at zero, ties to the lowest node index -- the reference's algorithm, order of
// operations and tolerances, in fp64.
//
// One warp per problem.  The cost matrix is either given (solve_emd) or formed
// in the kernel from the embedding rows exactly as pairwise_euclidean does it
// (fp64 norms and dots, (|a|^2 + |b|^2) - 2 a.b, clamp, sqrt, rounded once to
// f32; identical rows give exactly 0), and kept in shared memory next to the
// fp64 flow matrix and the per-node Dijkstra state.  Node scans are spread over the 32 lanes; the
// argmin is a warp reduction that keeps the lowest index on ties (np.argmin).
//
// Where the reference raises "no augmenting path" because float32-normalised
// supply and demand totals differ by more than 1e-9 (emd.py:153-162; about half
// of general histograms), augmentation stops once either side is exhausted.
#include <cfloat>

#include "common.cuh"

namespace lcrw {
namespace emd {

constexpr double kFeasTol = 1e-9;  // emd.py:33
constexpr int kMaxWarps = 8;

__host__ __device__ inline size_t problem_bytes(int h1, int h2) {
  const size_t n = (size_t)h1 + h2;
  // cost f64 [h1][h2], flow f64 [h1][h2], dist/phi/rem f64 [n], parent i32 [n], done u8 [n]
  const size_t b = (size_t)h1 * h2 * 16 + 3 * n * 8 + n * 4 + n;
  return (b + 15) / 16 * 16;
}

__device__ __forceinline__ void warp_argmin(double& v, int& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, off);
    const int oi = __shfl_xor_sync(0xffffffffu, i, off);
    if (ov < v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__global__ void __launch_bounds__(kMaxWarps * 32)
    emd_kernel(const double* __restrict__ supply, const int64_t* __restrict__ s_off, const double* __restrict__ demand,
               const int64_t* __restrict__ d_off, const double* __restrict__ costs, const int64_t* __restrict__ c_off,
               const float* __restrict__ E, int m, const int32_t* __restrict__ ids1, const int32_t* __restrict__ ids2,
               int64_t n_problems, size_t slot_bytes, double* __restrict__ objective, int32_t* __restrict__ status,
               double* __restrict__ flow_out, double* __restrict__ phi_out, uint8_t* __restrict__ gstate,
               int64_t prob_base) {
  extern __shared__ __align__(16) uint8_t emd_smem[];
  const int lane = threadIdx.x & 31;
  const int wip = threadIdx.x >> 5;
  const int64_t local = (int64_t)blockIdx.x * (blockDim.x >> 5) + wip;
  const int64_t prob = prob_base + local;
  if (prob >= n_problems) return;
  const int64_t a0 = s_off[prob], b0 = d_off[prob];
  const int h1 = (int)(s_off[prob + 1] - a0), h2 = (int)(d_off[prob + 1] - b0);
  const int n = h1 + h2;
  // state in shared memory, or -- for a problem too large for it -- in a global-memory
  // slot of the launch (same layout, same arithmetic; L1/L2 serve the scans)
  uint8_t* base = gstate ? gstate + (size_t)local * slot_bytes : emd_smem + (size_t)wip * slot_bytes;
  double* cost = reinterpret_cast<double*>(base);
  double* flow = cost + (size_t)h1 * h2;
  double* dist = flow + (size_t)h1 * h2;
  double* phi = dist + n;
  double* rem = phi + n;  // remaining supply (sources) / demand (sinks)
  int* parent = reinterpret_cast<int*>(rem + n);
  uint8_t* done = reinterpret_cast<uint8_t*>(parent + n);

  if (costs) {
    const double* cp = costs + c_off[prob];
    for (int c = lane; c < h1 * h2; c += 32) {
      cost[c] = cp[c];
      flow[c] = 0.0;
    }
  } else {
    // pairwise_euclidean(E[ids1], E[ids2]) (kernels.py:72-130), rounded once to f32 (emd.py:205)
    const int32_t* r1 = ids1 + a0;
    const int32_t* r2 = ids2 + b0;
    for (int i = lane; i < n; i += 32) {  // squared norms (fp64), parked in phi for now
      const float* row = E + (int64_t)(i < h1 ? r1[i] : r2[i - h1]) * m;
      double acc = 0.0;
      for (int d = 0; d < m; ++d) acc = fma((double)row[d], (double)row[d], acc);
      phi[i] = acc;
    }
    __syncwarp();
    for (int c = lane; c < h1 * h2; c += 32) {
      const int p = c / h2, q = c - p * h2;
      const float* ra = E + (int64_t)r1[p] * m;
      const float* rb = E + (int64_t)r2[q] * m;
      double dot = 0.0;
      for (int d = 0; d < m; ++d) dot = fma((double)ra[d], (double)rb[d], dot);
      const double sq = (phi[p] + phi[h1 + q]) - 2.0 * dot;
      cost[c] = (double)(float)sqrt(sq > 0.0 ? sq : 0.0);
      flow[c] = 0.0;
    }
  }
  for (int i = lane; i < n; i += 32) {
    phi[i] = 0.0;
    rem[i] = i < h1 ? supply[a0 + i] : demand[b0 + i - h1];
  }
  __syncwarp();

  // ---- successive shortest paths (emd.py:120-194) ----
  const int64_t max_rounds = 8ll * n * n + 64;
  int64_t rounds = 0;
  int st = 0;
  for (;;) {
    double rs = 0.0, rd = 0.0;
    for (int i = lane; i < n; i += 32) (i < h1 ? rs : rd) += rem[i];
    rs = warp_sum(rs);
    rd = warp_sum(rd);
    if (!(rs > kFeasTol) || !(rd > kFeasTol)) {
      if (rs > kFeasTol) st = 3;  // demand exhausted with supply left: the reference raises here
      break;
    }
    if (++rounds > max_rounds) {
      st = 2;
      break;
    }
    // multi-source Dijkstra over the residual network (emd.py:82-117)
    for (int i = lane; i < n; i += 32) {
      dist[i] = (i < h1 && rem[i] > kFeasTol) ? 0.0 : HUGE_VAL;
      parent[i] = -1;
      done[i] = 0;
    }
    __syncwarp();
    for (int it = 0; it < n; ++it) {
      double bv = HUGE_VAL;
      int bi = n;
      for (int i = lane; i < n; i += 32)
        if (!done[i] && dist[i] < bv) {
          bv = dist[i];
          bi = i;
        }
      warp_argmin(bv, bi);
      if (bi >= n || !(bv < HUGE_VAL)) break;
      const int u = bi;
      const double du = bv;
      if (lane == 0) done[u] = 1;
      __syncwarp();
      if (u < h1) {
        const double pu = phi[u];
        for (int q = lane; q < h2; q += 32) {
          const int v = h1 + q;
          if (done[v]) continue;
          double rc = (cost[u * h2 + q] + pu) - phi[v];
          rc = rc > 0.0 ? rc : 0.0;
          const double cand = du + rc;
          if (cand < dist[v]) {
            dist[v] = cand;
            parent[v] = u;
          }
        }
      } else {
        const int q = u - h1;
        const double pu = phi[u];
        for (int p = lane; p < h1; p += 32) {
          if (done[p] || !(flow[p * h2 + q] > kFeasTol)) continue;
          double rc = (pu - phi[p]) - cost[p * h2 + q];
          rc = rc > 0.0 ? rc : 0.0;
          const double cand = du + rc;
          if (cand < dist[p]) {
            dist[p] = cand;
            parent[p] = u;
          }
        }
      }
      __syncwarp();
    }
    // nearest sink with remaining demand
    double sv = HUGE_VAL;
    int t = n;
    for (int q = lane; q < h2; q += 32) {
      const double dq = rem[h1 + q] > kFeasTol ? dist[h1 + q] : HUGE_VAL;
      if (dq < sv) {
        sv = dq;
        t = q;
      }
    }
    warp_argmin(sv, t);
    if (!(sv < HUGE_VAL)) {
      st = 1;  // unbalanced beyond tolerance with both sides open
      break;
    }
    for (int i = lane; i < n; i += 32) phi[i] += dist[i] < sv ? dist[i] : sv;
    __syncwarp();
    if (lane == 0) {  // trace sink -> root, bottleneck, augment (sequential, path length <= n)
      int node = h1 + t;
      double bott = rem[h1 + t];
      while (parent[node] != -1) {
        const int prev = parent[node];
        if (node < h1) bott = fmin(bott, flow[node * h2 + (prev - h1)]);
        node = prev;
      }
      const int root = node;
      bott = fmin(bott, rem[root]);
      node = h1 + t;
      while (parent[node] != -1) {
        const int prev = parent[node];
        if (node >= h1)
          flow[prev * h2 + (node - h1)] += bott;
        else
          flow[node * h2 + (prev - h1)] -= bott;
        node = prev;
      }
      rem[root] -= bott;
      rem[h1 + t] -= bott;
    }
    __syncwarp();
  }
  double obj = 0.0;
  for (int c = lane; c < h1 * h2; c += 32) obj += flow[c] * cost[c];
  obj = warp_sum(obj);
  if (flow_out) {
    double* fo = flow_out + c_off[prob];
    for (int c = lane; c < h1 * h2; c += 32) fo[c] = flow[c];
  }
  if (phi_out) {  // potentials: sources at s_off, sinks after all sources (s_off[n_problems] + d_off)
    for (int i = lane; i < n; i += 32) {
      if (i < h1)
        phi_out[a0 + i] = phi[i];
      else
        phi_out[s_off[n_problems] + b0 + i - h1] = phi[i];
    }
  }
  if (lane == 0) {
    objective[prob] = obj;
#ifdef LCRW_EMD_ROUNDS
    status[prob] = st ? st : -(int)rounds;  // experiment build: augmentation count
#else
    status[prob] = st;
#endif
  }
}


// ---------------------------------------------------------------------------
// Small problems (h1 + h2 <= 32 * SLOTS): the per-node Dijkstra state lives in
// registers, node i in lane i % 32, slot i / 32.  The argmin is three integer
// warp reductions over the bit pattern of the (non-negative) distance and the
// node index -- the lexicographic (distance, index) minimum of np.argmin -- which
// is much shorter than a shuffle tree of doubles.  Same arithmetic as above.
// ---------------------------------------------------------------------------
template <int SLOTS, typename CT>  // CT: cost storage (float when formed in-kernel: the values are f32-rounded)
__global__ void __launch_bounds__(kMaxWarps * 32)
    emd_kernel_reg(const double* __restrict__ supply, const int64_t* __restrict__ s_off,
                   const double* __restrict__ demand, const int64_t* __restrict__ d_off,
                   const double* __restrict__ costs, const int64_t* __restrict__ c_off, const float* __restrict__ E,
                   int m, const int32_t* __restrict__ ids1, const int32_t* __restrict__ ids2, int64_t n_problems,
                   size_t slot_bytes, double* __restrict__ objective, int32_t* __restrict__ status,
                   double* __restrict__ flow_out, double* __restrict__ phi_out) {
  extern __shared__ __align__(16) uint8_t emd_smem[];
  const int lane = threadIdx.x & 31;
  const int wip = threadIdx.x >> 5;
  const int64_t prob = (int64_t)blockIdx.x * (blockDim.x >> 5) + wip;
  if (prob >= n_problems) return;
  const int64_t a0 = s_off[prob], b0 = d_off[prob];
  const int h1 = (int)(s_off[prob + 1] - a0), h2 = (int)(d_off[prob + 1] - b0);
  const int n = h1 + h2;
  uint8_t* base = emd_smem + (size_t)wip * slot_bytes;
  // shared: costs, a positive-flow bitmask (the only flow information the relaxations
  // need), potentials, parents; the fp64 flows themselves live in global memory
  // (flow_out layout) and are touched only along augmenting paths and at the end
  CT* cost = reinterpret_cast<CT*>(base);
  uint32_t* fmask = reinterpret_cast<uint32_t*>(base + ((size_t)h1 * h2 * sizeof(CT) + 7) / 8 * 8);
  double* phis = reinterpret_cast<double*>(fmask + (((size_t)h1 * h2 + 63) / 64) * 2);  // potentials
  double* flow = flow_out + c_off[prob];
  int* parent = reinterpret_cast<int*>(phis + n);     // written on relaxation, read by the path trace

  if (costs) {
    const double* cp = costs + c_off[prob];
    for (int c = lane; c < h1 * h2; c += 32) {
      cost[c] = (CT)cp[c];
      flow[c] = 0.0;
    }
    for (int w = lane; w < (h1 * h2 + 31) / 32; w += 32) fmask[w] = 0u;
  } else {
    const int32_t* r1 = ids1 + a0;
    const int32_t* r2 = ids2 + b0;
    for (int i = lane; i < n; i += 32) {
      const float* row = E + (int64_t)(i < h1 ? r1[i] : r2[i - h1]) * m;
      double acc = 0.0;
      for (int d = 0; d < m; ++d) acc = fma((double)row[d], (double)row[d], acc);
      phis[i] = acc;
    }
    __syncwarp();
    for (int c = lane; c < h1 * h2; c += 32) {
      const int p = c / h2, q = c - p * h2;
      const float* ra = E + (int64_t)r1[p] * m;
      const float* rb = E + (int64_t)r2[q] * m;
      double dot = 0.0;
      for (int d = 0; d < m; ++d) dot = fma((double)ra[d], (double)rb[d], dot);
      const double sq = (phis[p] + phis[h1 + q]) - 2.0 * dot;
      cost[c] = (CT)(float)sqrt(sq > 0.0 ? sq : 0.0);
      flow[c] = 0.0;
    }
    for (int w = lane; w < (h1 * h2 + 31) / 32; w += 32) fmask[w] = 0u;
    __syncwarp();
  }
  double phi[SLOTS], rem[SLOTS], dist[SLOTS];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) {
    const int i = lane + 32 * j;
    phi[j] = 0.0;
    rem[j] = i < h1 ? supply[a0 + i] : (i < n ? demand[b0 + i - h1] : 0.0);
    if (i < n) phis[i] = 0.0;
  }
  __syncwarp();

  const int64_t max_rounds = 8ll * n * n + 64;
  int64_t rounds = 0;
  int st = 0;
  for (;;) {
    double rs = 0.0, rd = 0.0;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const int i = lane + 32 * j;
      if (i < h1) rs += rem[j];
      else if (i < n) rd += rem[j];
    }
    rs = warp_sum(rs);
    rd = warp_sum(rd);
    if (!(rs > kFeasTol) || !(rd > kFeasTol)) {
      if (rs > kFeasTol) st = 3;  // demand exhausted with supply left: the reference raises here
      break;
    }
    if (++rounds > max_rounds) {
      st = 2;
      break;
    }
    uint32_t done = 0;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const int i = lane + 32 * j;
      dist[j] = (i < h1 && rem[j] > kFeasTol) ? 0.0 : HUGE_VAL;
      if (i < n) parent[i] = -1;
      if (i >= n) done |= 1u << j;
    }
    // sinks with remaining demand (warp-uniform bits): Dijkstra pops nodes in (distance,
    // index) order.  Once a sink with demand is popped at distance sv, every node not yet
    // popped has a final distance >= sv, so min(dist, sv) (the potential update) is already
    // final.  The reference's argmin picks the LOWEST-index sink at distance sv, which may
    // only reach sv through zero-reduced-cost arcs of nodes popped later at the same
    // distance, so the search goes on while the popped distance equals sv (bitwise) and
    // stops at the first larger one: same sink, same parents, same potentials as the
    // full search (emd.py:104-129, 166-170)
    uint32_t dmask[SLOTS];
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const int i = lane + 32 * j;
      dmask[j] = __ballot_sync(0xffffffffu, i >= h1 && i < n && rem[j] > kFeasTol);
    }
    int t_hit = -1;
    double sv_hit = HUGE_VAL;
    __syncwarp();
    for (int it = 0; it < n; ++it) {
      double bv = HUGE_VAL;
      int bi = 0x7FFFFFFF;
#pragma unroll
      for (int j = 0; j < SLOTS; ++j)
        if (!((done >> j) & 1u) && dist[j] < bv) {
          bv = dist[j];
          bi = lane + 32 * j;
        }
      // lexicographic (distance, index) minimum: non-negative doubles order like their bits
      const uint32_t hi = (uint32_t)__double2hiint(bv);
      const uint32_t mhi = __reduce_min_sync(0xffffffffu, hi);
      const uint32_t lo = hi == mhi ? (uint32_t)__double2loint(bv) : 0xFFFFFFFFu;
      const uint32_t mlo = __reduce_min_sync(0xffffffffu, lo);
      const uint32_t ix = (hi == mhi && lo == mlo) ? (uint32_t)bi : 0xFFFFFFFFu;
      const int u = (int)__reduce_min_sync(0xffffffffu, ix);
      const double du = __hiloint2double((int)mhi, (int)mlo);
      if (u >= n || !(du < HUGE_VAL)) break;
      if (t_hit >= 0 && du != sv_hit) break;  // every node at the hit distance is popped
      {
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < SLOTS; ++j) w = (u >> 5) == j ? dmask[j] : w;
        if (((w >> (u & 31)) & 1u) && (t_hit < 0 || u - h1 < t_hit)) {
          t_hit = u - h1;
          sv_hit = du;
        }
      }
      if (lane == (u & 31)) done |= 1u << (u >> 5);
      const double pu = phis[u];
      if (u < h1) {
        const CT* crow = cost + u * h2;
#pragma unroll
        for (int j = 0; j < SLOTS; ++j) {
          const int v = lane + 32 * j;
          if (v < h1 || v >= n || ((done >> j) & 1u)) continue;
          double rc = ((double)crow[v - h1] + pu) - phi[j];
          rc = rc > 0.0 ? rc : 0.0;
          const double cand = du + rc;
          if (cand < dist[j]) {
            dist[j] = cand;
            parent[v] = u;
          }
        }
      } else {
        const int q = u - h1;
#pragma unroll
        for (int j = 0; j < SLOTS; ++j) {
          const int pn = lane + 32 * j;
          const int cell = pn * h2 + q;
          if (pn >= h1 || ((done >> j) & 1u) || !((fmask[cell >> 5] >> (cell & 31)) & 1u)) continue;
          double rc = (pu - phi[j]) - (double)cost[pn * h2 + q];
          rc = rc > 0.0 ? rc : 0.0;
          const double cand = du + rc;
          if (cand < dist[j]) {
            dist[j] = cand;
            parent[pn] = u;
          }
        }
      }
    }
    // nearest sink with remaining demand
    double sv = HUGE_VAL;
    int t = 0x7FFFFFFF;
    if (t_hit >= 0) {
      sv = sv_hit;
      t = t_hit;
    } else {
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const int i = lane + 32 * j;
      if (i >= h1 && i < n && rem[j] > kFeasTol && dist[j] < sv) {
        sv = dist[j];
        t = i - h1;
      }
    }
    {
      const uint32_t hi = (uint32_t)__double2hiint(sv);
      const uint32_t mhi = __reduce_min_sync(0xffffffffu, hi);
      const uint32_t lo = hi == mhi ? (uint32_t)__double2loint(sv) : 0xFFFFFFFFu;
      const uint32_t mlo = __reduce_min_sync(0xffffffffu, lo);
      const uint32_t ix = (hi == mhi && lo == mlo) ? (uint32_t)t : 0xFFFFFFFFu;
      t = (int)__reduce_min_sync(0xffffffffu, ix);
      sv = __hiloint2double((int)mhi, (int)mlo);
    }
    }
    if (!(sv < HUGE_VAL)) {
      st = 1;
      break;
    }
    __syncwarp();  // every lane's Dijkstra reads of phis precede the potential update (WAR)
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const int i = lane + 32 * j;
      phi[j] += dist[j] < sv ? dist[j] : sv;
      if (i < n) phis[i] = phi[j];
    }
    __syncwarp();
    // path trace (lane 0) -> bottleneck -> augment; remaining amounts live in registers,
    // so the root and sink updates are applied by their owner lanes afterwards
    int root = 0;
    double bott = 0.0;
    const int sink = h1 + t;
    double rem_sink = 0.0;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const double r = __shfl_sync(0xffffffffu, rem[j], sink & 31);
      if ((sink >> 5) == j) rem_sink = r;
    }
    if (lane == 0) {
      int node = sink;
      bott = rem_sink;
      while (parent[node] != -1) {
        const int prev = parent[node];
        if (node < h1) bott = fmin(bott, flow[node * h2 + (prev - h1)]);
        node = prev;
      }
      root = node;
    }
    root = __shfl_sync(0xffffffffu, root, 0);
    double rem_root = 0.0;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const double r = __shfl_sync(0xffffffffu, rem[j], root & 31);
      if ((root >> 5) == j) rem_root = r;
    }
    if (lane == 0) {
      bott = fmin(bott, rem_root);
      int node = sink;
      while (parent[node] != -1) {
        const int prev = parent[node];
        const int cell = node >= h1 ? prev * h2 + (node - h1) : node * h2 + (prev - h1);
        const double f = node >= h1 ? flow[cell] + bott : flow[cell] - bott;
        flow[cell] = f;
        const uint32_t bit = 1u << (cell & 31);
        fmask[cell >> 5] = f > kFeasTol ? (fmask[cell >> 5] | bit) : (fmask[cell >> 5] & ~bit);
        node = prev;
      }
    }
    bott = __shfl_sync(0xffffffffu, bott, 0);
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const int i = lane + 32 * j;
      if (i == root) rem[j] -= bott;
      if (i == sink) rem[j] -= bott;
    }
    __syncwarp();
  }
  double obj = 0.0;
  for (int c = lane; c < h1 * h2; c += 32) obj += flow[c] * (double)cost[c];
  obj = warp_sum(obj);

  if (phi_out) {
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const int i = lane + 32 * j;
      if (i < h1)
        phi_out[a0 + i] = phi[j];
      else if (i < n)
        phi_out[s_off[n_problems] + b0 + i - h1] = phi[j];
    }
  }
  if (lane == 0) {
    objective[prob] = obj;
#ifdef LCRW_EMD_ROUNDS
    status[prob] = st ? st : -(int)rounds;
#else
    status[prob] = st;
#endif
  }
}

}  // namespace emd
}  // namespace lcrw

using namespace lcrw;
using namespace lcrw::emd;

extern "C" {

size_t lcrw_emd_problem_bytes(int h1, int h2) { return problem_bytes(h1, h2); }

static size_t problem_bytes_reg(int h1, int h2, size_t cost_bytes) {
  const size_t n = (size_t)h1 + h2;
  const size_t c = ((size_t)h1 * h2 * cost_bytes + 7) / 8 * 8;
  const size_t mask = ((size_t)h1 * h2 + 63) / 64 * 8;
  const size_t b = c + mask + n * 8 + n * 4;  // cost, positive-flow bits, phi, parent (flows: global)
  return (b + 15) / 16 * 16;
}

int lcrw_emd_batch(const double* supply, const int64_t* s_off, const double* demand, const int64_t* d_off,
                   const double* costs, const int64_t* c_off, const float* E, int64_t v, int m, const int32_t* ids1,
                   const int32_t* ids2, int64_t n_problems, int max_h1, int max_h2, double* objective,
                   int32_t* status, double* flow_out, double* phi_out, void* stream) {
  LCRW_REQUIRE(n_problems >= 0, "lcrw_emd_batch: bad shape");
  if (n_problems == 0) return LCRW_OK;
  LCRW_REQUIRE(supply && s_off && demand && d_off && objective && status, "lcrw_emd_batch: null pointer");
  LCRW_REQUIRE(costs ? (c_off != nullptr) : (E && ids1 && ids2 && m > 0 && v > 0),
               "lcrw_emd_batch: need either explicit costs (+ c_off) or embeddings and word ids");
  LCRW_REQUIRE(!flow_out || c_off, "lcrw_emd_batch: flow_out needs c_off");
  LCRW_REQUIRE(max_h1 >= 1 && max_h2 >= 1, "lcrw_emd_batch: every histogram needs at least one word");
  const int nmax = max_h1 + max_h2;
  const int slots = nmax <= 32 ? 1 : nmax <= 64 ? 2 : nmax <= 96 ? 3 : nmax <= 128 ? 4 : 0;
  const size_t slot = slots ? problem_bytes_reg(max_h1, max_h2, costs ? 8 : 4) : problem_bytes(max_h1, max_h2);
  const size_t smem_max = 227 * 1024;
  cudaStream_t st = as_stream(stream);
  if (slot > smem_max) {
    // too large for shared memory: the general kernel with its per-problem state in global
    // memory, one warp per block, in launches of at most kGlobalProblems problems
    constexpr int64_t kGlobalProblems = 4096;
    const int64_t per = n_problems < kGlobalProblems ? n_problems : kGlobalProblems;
    uint8_t* gstate = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&gstate), (size_t)per * slot, st);
    if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync(emd global state)");
    ProfScope prof(st, "emd_global");
    for (int64_t p0 = 0; p0 < n_problems; p0 += per) {
      const int64_t cnt = n_problems - p0 < per ? n_problems - p0 : per;
      emd_kernel<<<(unsigned)cnt, 32, 0, st>>>(supply, s_off, demand, d_off, costs, c_off, E, m, ids1, ids2,
                                               n_problems, slot, objective, status, flow_out, phi_out, gstate, p0);
      LCRW_CHECK_LAUNCH("emd_kernel (global state)");
    }
    e = cudaFreeAsync(gstate, st);
    if (e != cudaSuccess) return cuda_status(e, "cudaFreeAsync(emd global state)");
    return LCRW_OK;
  }
  // one problem (warp) per block by default: a block's shared memory is one slot, so an
  // SM holds as many problems as their slots allow (up to 32 blocks) instead of one
  // block of kMaxWarps slots
#ifndef LCRW_EMD_WPB
#define LCRW_EMD_WPB 1
#endif
  int warps = (int)(smem_max / slot);
  if (warps > LCRW_EMD_WPB) warps = LCRW_EMD_WPB;
  const size_t smem = slot * warps;
  static bool attr = false;
  if (!attr) {
    const void* fns[9] = {(const void*)emd_kernel,
                          (const void*)emd_kernel_reg<1, double>, (const void*)emd_kernel_reg<2, double>,
                          (const void*)emd_kernel_reg<3, double>, (const void*)emd_kernel_reg<4, double>,
                          (const void*)emd_kernel_reg<1, float>,  (const void*)emd_kernel_reg<2, float>,
                          (const void*)emd_kernel_reg<3, float>,  (const void*)emd_kernel_reg<4, float>};
    for (const void* f : fns) {
      cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(emd kernels)");
    }
    attr = true;
  }
  const int64_t blocks = (n_problems + warps - 1) / warps;
  LCRW_REQUIRE(blocks < (1ll << 31), "lcrw_emd_batch: too many problems");
  LCRW_REQUIRE(!slots || c_off, "lcrw_emd_batch: c_off (per-problem h1*h2 offsets) is required");
  // the register-state kernels keep flows in global memory (flow_out layout): without a
  // caller buffer, a stream-ordered scratch one sized for the largest problem each
  double* scratch = nullptr;
  if (slots && !flow_out) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                                    (size_t)n_problems * max_h1 * max_h2 * sizeof(double), st);
    if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync(emd flow scratch)");
    flow_out = scratch;
  }
  ProfScope prof(st, "emd");
#define LCRW_EMD_LAUNCH(K, ...)                                                                                 \
  K<<<(unsigned)blocks, warps * 32, smem, st>>>(supply, s_off, demand, d_off, costs, c_off, E, m, ids1, ids2,   \
                                               n_problems, slot, objective, status, flow_out, phi_out __VA_ARGS__)
  if (costs) {
    switch (slots) {
      case 1: LCRW_EMD_LAUNCH((emd_kernel_reg<1, double>)); break;
      case 2: LCRW_EMD_LAUNCH((emd_kernel_reg<2, double>)); break;
      case 3: LCRW_EMD_LAUNCH((emd_kernel_reg<3, double>)); break;
      case 4: LCRW_EMD_LAUNCH((emd_kernel_reg<4, double>)); break;
      default: LCRW_EMD_LAUNCH(emd_kernel, , nullptr, 0); break;
    }
  } else {
    switch (slots) {
      case 1: LCRW_EMD_LAUNCH((emd_kernel_reg<1, float>)); break;
      case 2: LCRW_EMD_LAUNCH((emd_kernel_reg<2, float>)); break;
      case 3: LCRW_EMD_LAUNCH((emd_kernel_reg<3, float>)); break;
      case 4: LCRW_EMD_LAUNCH((emd_kernel_reg<4, float>)); break;
      default: LCRW_EMD_LAUNCH(emd_kernel, , nullptr, 0); break;
    }
  }
#undef LCRW_EMD_LAUNCH
  LCRW_CHECK_LAUNCH("emd_kernel");
  if (scratch) {
    cudaError_t e = cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return cuda_status(e, "cudaFreeAsync(emd flow scratch)");
  }
  return LCRW_OK;
}

}  // extern "C"
