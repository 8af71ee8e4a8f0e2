// ipm_kernels.cuh — the persistent per-problem IPM kernels (solve: init +
// Alg. 1; backward: Alg. 2 + Alg. 3) and the batch-sum kernels for gradients
// of shared parameters.  One CTA owns one QP for the whole kernel; the KKT
// matrix, the iterate and all per-iteration vectors live in shared memory;
// the problem data (Q, G, A, …) is re-read from global memory (L1/L2) each
// iteration.  DESIGN.md §5 (layout) and §6 (roofline).
//
// Linear system (readings Q12 + Q12b).  Each Newton step solves
// the bounded system of Eq. 14.  It is first brought to the
// congruent quasi-definite form M (Δv = GΔx + w), then every w_i of a
// constraint with v_i ≤ 0 is eliminated exactly (its pivot is −d₋_i with
// d₋_i ≥ ½).  The factored matrix is
//     [[Q + Gᵀ diag(ω) G,  G_Aᵀ D₊_A,  Aᵀ],
//      [D₊_A G_A,          −D₋_A,      0 ],
//      [A,                  0,          0 ]]
// with A = {i : v_i > 0} and ω_i = d₊_i on A, ω_i = d₊_i/d₋_i = b(v_i)/b(−v_i) ≤ 1
// off A: every entry stays bounded (the property the paper's method rests
// on), and the size drops from n+p+m to n+|A|+m.
#pragma once
#include <type_traits>

#include "ipm_cta.cuh"
#include "tc_factor.cuh"
#include "tc_syrk.cuh"

namespace qpb {

enum { ST_CONVERGED = 0, ST_MAX_ITER = 2, ST_FAIL = 3 };
enum { STG_SCALING = 1, STG_PREDICTOR = 2, STG_CENTERING = 3, STG_CORRECTOR = 4, STG_LINESEARCH = 5,
       STG_RELAX = 6, STG_BACKWARD = 7, STG_INIT = 8 };

struct Args {
  int B, n, m, p;
  int n4, Nmax, N4max;   // KKT capacity: N ≤ n4 + p + m
  int ksmem, ncap;       // shared-memory KKT buffer (floats) and the largest N it holds
  long long kglob_size;  // floats per global KKT workspace (worst case N)
  const float *Q, *q, *A, *b, *G, *h;
  long long sQ, sq, sA, sb, sG, sh;
  float *x, *y, *z, *s;  // solution (solve: out; backward: in)
  int *iters, *status;
  const float* dl;
  float *gQ, *gq, *gA, *gb, *gG, *gh;     // per-problem gradients (nullptr = skip)
  float *wx, *wy, *wz, *wdx, *wdy, *wdz;  // per-problem vectors for shared sums (nullptr = skip)
  int *riters, *rstatus;
  float tol, sigma, tau, kappa_relax, relax_ktol, floor_rel, relax_tol;
  int max_iter, relax_max_iter;
  unsigned long long* prof;  // optional per-CTA phase cycle counters (diagnostics; nullptr = off)
  float* flops;              // per-problem algorithmic flops of this call, nullptr = off
  float* kglob;              // per-CTA KKT workspaces in global memory (iterations with N > ncap)
  int tcf;                   // floats of the tensor-core staging area (large-N kernels; 0 = none)
  int rof;                   // entries of the row-offset table (path 1: N4max; 0 = none)
  int pcap;                  // largest |A| the KKT buffer holds (reading Q12c; p = no cap)
  int* sched;                // problem counter of this launch (dynamic assignment; zeroed by the host)
  int* done;                 // per problem: epoch of the last solve that finished it
  int epoch;                 // this solve's epoch (backward: the solve it differentiates)
  int* status_out;           // solve: second copy of the status (the caller's array), nullptr = none
  unsigned long long* tl;    // diagnostics (QPB200_TIMELINE): per problem {smid, t_start, t_end} (ns)
  int bwd;                   // 0: solve launch (init + Alg. 1), 1: backward launch (Alg. 2 + Alg. 3)
  // Reading Q12c guard (path 1): a problem whose capped elimination would put
  // a weight ω > fb_bound on an eliminated v_i > 0 constraint is handed to the
  // uncapped large-N kernel (the fallback launch that follows on the stream)
  float fb_bound;            // 0 = no check (large-N kernels, uncapped)
  int* fb_flag;              // [B] solve: 1 = handed over (read by the backward)
  int* fb_list;              // this call's hand-over list (chunk-local problem indices)
  int* fb_count;             // its length
  const int* plist;          // list-driven launch (the fallback): problems plist[i], i < *pcount
  const int* pcount;
  // Guarded chord relax (reading Q26): the
  // solve caches the factorisation of its first iterate with κ < √10·κ_relax
  // (the factor, its pivot reciprocals and the Jacobian vectors it was built
  // from); the backward takes chord steps on it while they contract
  int relax_mode;            // 0: exact Newton (Q6); 2: guarded chord
  int chord_max;             // most chord steps per problem
  float chord_rho;           // contraction a chord step must reach
  float* kc;                 // [B][kc_stride] cached factors (nullptr = no chord)
  long long kc_stride;
  float* chd;                // [B][chd_stride] cached Jacobian: {pa, κ, ·, ·}, d₊[p4], d₋[p4], c[p4], widx[p4], rinv[N4max]
  long long chd_stride;
  int* chord_ok;             // [B] 1 = this problem's solve cached a factor
  int* chord_cnt;            // backward: chord steps taken, summed over the batch (path 1)
};

// chord cache block of one problem (floats): 4 scalars, then d₊, d₋, c, widx, rinv
__host__ __device__ inline long long chd_floats(int p, int N4max) {
  const int p4 = (p + 3) & ~3;
  return 4 + 4LL * p4 + ((N4max + 3) & ~3);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// griddepcontrol.wait: block until every grid this launch depends on
// (programmatic stream serialisation) has completed and its memory is
// visible; returns at once when the launch has no such dependency.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

// Next problem for this CTA: problems are handed out in increasing order as
// CTAs free up (one atomic per problem), so a CTA that drew short problems
// takes more of them.  Block-uniform.
__device__ __forceinline__ int next_problem(const Args& a, int* slot) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int i = atomicAdd(a.sched, 1);
    *slot = !a.plist ? i : (i < *a.pcount ? a.plist[i] : a.B);  // the fallback walks its list
  }
  __syncthreads();
  return *slot;
}

// Algorithmic flops of one Newton iteration on the reduced system of size
// Nr = n + |A| + m: assembly p·n(n+1) + |A|·n, factorisation
// Nr³/3, two triangular solves 2·Nr², residual GEMVs 2n² + 6pn + 4mn,
// Δv recovery 2pn.
__device__ __forceinline__ float iter_flops(int n, int m, int p, int pa, bool resid, bool fac, bool solve) {
  const float Nr = (float)(n + pa + m);
  float f = 0.f;
  if (resid) f += 2.f * n * n + 6.f * p * n + 4.f * m * n;
  if (fac) f += (float)p * n * (n + 1) + (float)pa * n + Nr * Nr * Nr / 3.f;
  if (solve) f += 2.f * Nr * Nr + 2.f * p * n;
  return f;
}

// Shared-memory carve-up (floats).  Every segment is a multiple of 4 floats
// so that float4 accesses stay 16-byte aligned.  layout() sizes the
// allocation on the host (base = nullptr) and carves it on the device.
struct Smem {
  float *K, *rinv, *rhs;
  float *x, *y, *z, *s, *v, *dp, *dm, *c, *om;
  float *rz, *rs, *f2, *t, *gx, *dx, *dy, *dz, *ds_x;
  float *red, *scr, *colscr;
  int *act, *widx, *flag;
  float* tc;  // tcgen05 operand staging + mbarrier (large-N kernels)
  int* ro;    // row offsets of this iteration's KKT layout (path 1; N4max entries)
  float* end;
};

__host__ __device__ inline Smem layout(float* base, int n4, int m, int p, int N4max, int ksize, int tcf, int rof) {
  const int m4 = (m + 3) & ~3, p4 = (p + 3) & ~3;
  Smem S;
  float* q = base;
  S.K = q; q += ksize;
  S.rinv = q; q += N4max;
  S.rhs = q; q += N4max;
  S.x = q; q += n4;
  S.y = q; q += m4;
  S.z = q; q += p4;
  S.s = q; q += p4;
  S.v = q; q += p4;
  S.dp = q; q += p4;
  S.dm = q; q += p4;
  S.c = q; q += p4;
  S.om = q; q += p4;
  S.rz = q; q += p4;
  S.rs = q; q += p4;
  S.f2 = q; q += p4;
  S.t = q; q += p4;
  S.gx = q; q += p4 + m4;
  S.dx = q; q += n4;
  S.dy = q; q += m4;
  S.dz = q; q += p4;
  S.ds_x = q; q += n4 + m4;  // standard arm: predictor / centering Δx, Δy
  S.red = q; q += 160;
  S.scr = q; q += 16 * 17 + 16;
  // residual column partial sums (≤ 4 groups × 4 sums × 64 columns): used only
  // inside residuals(), while the KKT buffer holds nothing live (the previous
  // factor was consumed by its solve; the next assembly follows), so they
  // alias the buffer when it is large enough
  if (ksize >= 4 * 4 * 64) {
    S.colscr = S.K;
  } else {
    S.colscr = q; q += 4 * 4 * 64;
  }
  S.act = reinterpret_cast<int*>(q); q += p4;
  S.widx = reinterpret_cast<int*>(q); q += p4;
  S.flag = reinterpret_cast<int*>(q); q += 16;
  S.tc = q; q += tcf;
  S.ro = reinterpret_cast<int*>(q); q += (rof + 3) & ~3;
  S.end = q;
  return S;
}

__host__ inline size_t ipm_smem_bytes(int n4, int m, int p, int N4max, int ksize, int tcf, int rof) {
  const Smem S = layout(nullptr, n4, m, p, N4max, ksize, tcf, rof);
  return (size_t)reinterpret_cast<uintptr_t>(S.end);
}

__device__ inline Smem carve(float* base, const Args& a) {
  return layout(base, a.n4, a.m, a.p, a.N4max, a.ksmem, a.tcf, a.rof);
}

// Where this iteration's KKT matrix lives.  Path 1 kernels (BIG = false)
// always use the shared-memory buffer (the host guarantees it holds the
// worst case), so the compiler emits shared-memory instructions; the large-N
// kernels choose at run time: the smem buffer when the reduced system fits
// (N ≤ ncap), else the CTA's global workspace (L2).
template <bool BIG>
__device__ __forceinline__ float* kkt_ptr(const Smem& S, const Args& a, const KLayout& L) {
  if (!BIG) return S.K;
  return L.N <= a.ncap ? S.K : a.kglob + (size_t)blockIdx.x * (size_t)a.kglob_size;
}

// factor_qd keeps up to 256/NT panel rows per thread in registers; larger
// systems stream their panel rows (factor_big).
// floats of the shared-memory KKT buffer (it ends where rinv starts)
__device__ __forceinline__ int ksmem_of(const Smem& S) { return (int)(S.rinv - S.K); }

template <int NT, bool BIG, int MAXN4 = 256>
__device__ __forceinline__ int factor_any(float* K, const Smem& S, const KLayout& L, float theta) {
  if constexpr (BIG) {
    // large N: tensor-core left-looking panels (QPB200_NO_TC_FACTOR: FP32 factor_big, for A/B)
#ifndef QPB200_NO_TC_FACTOR
    if (L.N4 > 256)  // K lives in the global workspace: the smem KKT buffer stages the panels
      return factor_tc<NT>(K, L, theta, S.rinv, S.flag, S.scr, tc::tc_state(S.tc), K == S.K ? nullptr : S.K,
                           K == S.K ? 0 : ksmem_of(S));
#else
    if (L.N4 > 256) return factor_big<NT>(K, L, theta, S.rinv, S.flag, S.scr);
#endif
  }
  if constexpr (BIG) return factor_qd<NT>(K, L, theta, S.rinv, S.flag, S.scr);
  else return factor_qd<NT, true, MAXN4>(K, L, theta, S.rinv, S.flag, S.scr, S.ro);
}

struct Prob {
  const float *Q, *q, *A, *b, *G, *h;
};

__device__ __forceinline__ Prob prob_of(const Args& a, int bid) {
  Prob P;
  P.Q = a.Q + a.sQ * bid; P.q = a.q + a.sq * bid; P.A = a.A + a.sA * bid;
  P.b = a.b + a.sb * bid; P.G = a.G + a.sG * bid; P.h = a.h + a.sh * bid;
  return P;
}

// ------------------------------------------------------------------------
// Active-set compaction: act[0..pa) = the kept constraints in increasing
// order, widx[k] = position in act or −1.  Returns pa (block-uniform).
// Kept = {k : v_k > 0} (reading Q12b); when that set is larger than pcap
// (reading Q12c: the shared-memory KKT buffer of this kernel holds at most
// n4 + pcap + m rows), only the pcap constraints with the LARGEST v_k are
// kept (ties: smaller k first) and the others are eliminated like those with
// v_k ≤ 0, with weight ω_k = d₊/d₋.
// ------------------------------------------------------------------------
template <int NT, class Pred>
__device__ int compact_pass(const Smem& S, int p, Pred on_of) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int base = 0;
  for (int c0 = 0; c0 < p; c0 += NT) {
    const int k = c0 + tid;
    const bool on = k < p && on_of(k);
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    __syncthreads();
    if (lane == 0) S.flag[warp] = __popc(bal);  // NW ≤ 16 counters
    __syncthreads();
    int before = base;
    for (int w = 0; w < warp; ++w) before += S.flag[w];
    int tot = 0;
    for (int w = 0; w < NW; ++w) tot += S.flag[w];
    if (k < p) {
      const int pos = before + __popc(bal & ((1u << lane) - 1u));
      S.widx[k] = on ? pos : -1;
      if (on) S.act[pos] = k;
    }
    base += tot;
  }
  __syncthreads();
  return base;
}

template <int NT>
__device__ int compact_active(const Smem& S, int p, bool all_inactive, int pcap, bool* capped = nullptr) {
  if (capped) *capped = false;
  if (all_inactive) return compact_pass<NT>(S, p, [](int) { return false; });
  const float* v = S.v;
  const int pa = compact_pass<NT>(S, p, [v](int k) { return v[k] > 0.f; });
  if (pa <= pcap) return pa;
  if (capped) *capped = true;
  return compact_pass<NT>(S, p, [v, p, pcap](int k) {
    const float vk = v[k];
    if (!(vk > 0.f)) return false;
    int rank = 0;  // constraints ordered before k: larger v, or equal v and smaller index
    for (int j = 0; j < p; ++j) rank += (v[j] > vk || (v[j] == vk && j < k)) ? 1 : 0;
    return rank < pcap;
  });
}

// ------------------------------------------------------------------------
// KKT assembly of the reduced bounded system (header comment), lower triangle
// in the packed layout L (N = n4 + pa + m).  cw = weights of the C rows (d₊),
// e = the −diagonal of the w block (d₋), om = ω.  Returns max|diag|.
// ------------------------------------------------------------------------
template <int NT, bool TC = false>
__device__ float assemble(float* K, const Smem& S, const Args& a, const Prob& P, const KLayout& L, int pa,
                          const float* om, const float* cw, const float* e) {
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, N = L.N, N4 = L.N4;
  // 1. zero the whole buffer of this layout (float4 stores), then scatter the
  //    nonzeros of the rows ≥ n4: C rows d₊_k g_k of the active constraints,
  //    A rows, −d₋ on the w diagonal, −1 on padding rows.
  if constexpr (!TC)  // row-offset table of this layout (path 1), read after the barrier below
    for (int i = tid; i < L.N4; i += NT) S.ro[i] = L.off(i);
  {
    // (the tensor-core epilogue writes every stored entry of rows < n4 itself)
    float4* K4 = reinterpret_cast<float4*>(K);
    const int nz4 = L.size() >> 2;
    const int z0 = !TC ? 0 : (n4 < L.N4 ? L.off(n4) >> 2 : nz4);
    for (int i = z0 + tid; i < nz4; i += NT) K4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  const int nrow = N - n4;  // C rows then A rows
  const bool pairs = !TC && !(n & 1) &&
                     !((reinterpret_cast<uintptr_t>(P.G) | (a.m > 0 ? reinterpret_cast<uintptr_t>(P.A) : 0)) & 7);
  if (pairs) {
    // even n (path 1): column pairs, float2 loads and stores (rows of K start
    // at multiples of 4 floats)
    const int n2 = n >> 1, tot = nrow * n2;
    const int drr = NT / n2, dj = NT - drr * n2;
    int rr = tid / n2, jp = tid - rr * n2;
    for (int idx = tid; idx < tot; idx += NT) {
      float2 val;
      if (rr < pa) {
        const int k = S.act[rr];
        const float w = cw[k];
        val = __ldg(reinterpret_cast<const float2*>(P.G + k * n) + jp);
        val.x *= w; val.y *= w;
      } else {
        val = __ldg(reinterpret_cast<const float2*>(P.A + (rr - pa) * n) + jp);
      }
      *reinterpret_cast<float2*>(K + row_off<!TC>(L, S.ro, n4 + rr) + 2 * jp) = val;
      rr += drr; jp += dj;
      if (jp >= n2) { jp -= n2; ++rr; }
    }
  } else {
    // large n: 4 elements per thread and step, loads issued before the stores
    // (path 1 keeps one: measured 1.5 % faster there)
    constexpr int UB = TC ? 4 : 1;
    const int tot = nrow * n;
    // (row, column) of this thread's element, advanced by NT elements per
    // step without a division: NT = drr rows + dj columns
    const int drr = NT / n, dj = NT - drr * n;
    int rr = tid / n, j = tid - rr * n;
    for (int base = 0; base < tot; base += UB * NT) {
      float val[UB];
      int dst[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int idx = base + u * NT + tid;
        dst[u] = -1;
        val[u] = 0.f;
        if (idx < tot) {
          if (rr < pa) {
            const int k = S.act[rr];
            val[u] = cw[k] * __ldg(P.G + k * n + j);
          } else {
            val[u] = __ldg(P.A + (rr - pa) * n + j);
          }
          dst[u] = row_off<!TC>(L, S.ro, n4 + rr) + j;
        }
        rr += drr; j += dj;
        if (j >= n) { j -= n; ++rr; }
      }
#pragma unroll
      for (int u = 0; u < UB; ++u)
        if (dst[u] >= 0) K[dst[u]] = val[u];
    }
  }
  for (int r = n4 + tid; r < N4; r += NT)
    K[row_off<!TC>(L, S.ro, r) + r] = r < n4 + pa ? -e[S.act[r - n4]] : (r < N ? 0.f : -1.f);
  float dmax = 0.f;
  if constexpr (TC) {
    // 2'. large n: H = Q + Gᵀ diag(ω) G on the tensor cores (tc_syrk.cuh,
    //     3×TF32), 128×128 tiles of the lower triangle; the epilogue adds Q
    //     (identity on the padding rows n..n4) and stores the lower part.
    const tc::TcState ts = tc::tc_state(S.tc);
    for (int i0 = 0; i0 < n4; i0 += tc::TM)
      for (int j0 = 0; j0 <= i0; j0 += tc::TN)
        tc::syrk_tile<NT>(ts, P.G, om, p, n, i0, j0, [&](int row0, int j, const float* t) {
          float qv[32];  // all 32 Q loads in flight before the first use
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const int i = row0 + r;
            qv[r] = (i < n && j < n && j <= i) ? __ldg(P.Q + (size_t)i * n + j) : 0.f;
          }
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const int i = row0 + r;
            if (i < n4 && j <= i) {
              const float val = (i < n && j < n) ? qv[r] + t[33 * r] : (i == j ? 1.f : 0.f);
              K[L.off(i) + j] = val;
              if (i == j && i < n) dmax = fmaxf(dmax, fabsf(val));
            }
          }
        });
  } else {
  // 2. H = Q + Gᵀ diag(ω) G: 4×4 register tiles of the lower triangle; G rows
  //    are read from global memory (L1-resident across iterations).
  const int T = n4 >> 2;
  const int nt = T * (T + 1) / 2;
  for (int t = tid; t < nt; t += NT) {
    int I = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    const int J = t - I * (I + 1) / 2;
    const int i0 = 4 * I, j0 = 4 * J;
    float acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int i = i0 + u, j = j0 + w;
        acc[u][w] = (i < n && j < n) ? __ldg(P.Q + i * n + j) : (i == j ? 1.f : 0.f);
      }
    // 4 rows of G in flight per step (loads issued before the FMAs); for even
    // n the rows are 8-byte aligned and each 4-wide strip is two float2 loads
    auto kloop = [&](auto even_t) {
      constexpr bool EVEN = decltype(even_t)::value;
      auto ld4 = [&](const float* g, int c0, float (&o)[4]) {
        if constexpr (EVEN) {  // c0 % 4 == 0, n even: c0 < n ⇒ c0 + 1 < n
          const float2 a = c0 < n ? __ldg(reinterpret_cast<const float2*>(g + c0)) : make_float2(0.f, 0.f);
          const float2 b = c0 + 2 < n ? __ldg(reinterpret_cast<const float2*>(g + c0 + 2)) : make_float2(0.f, 0.f);
          o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) o[u] = c0 + u < n ? __ldg(g + c0 + u) : 0.f;
        }
      };
      int k = 0;
      for (; k + 4 <= p; k += 4) {
        float gi[4][4], gj[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* g = P.G + (k + q) * n;
          ld4(g, i0, gi[q]);
          ld4(g, j0, gj[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float w = om[k + q];
#pragma unroll
          for (int u = 0; u < 4; ++u) gj[q][u] *= w;
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int w2 = 0; w2 < 4; ++w2) acc[u][w2] = fmaf(gi[q][u], gj[q][w2], acc[u][w2]);
        }
      }
      for (; k < p; ++k) {
        const float* g = P.G + k * n;
        const float w = om[k];
        float gi[4], gj[4];
        ld4(g, i0, gi);
        ld4(g, j0, gj);
#pragma unroll
        for (int u = 0; u < 4; ++u) gj[u] *= w;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int w2 = 0; w2 < 4; ++w2) acc[u][w2] = fmaf(gi[u], gj[w2], acc[u][w2]);
      }
    };
    if ((n & 1) == 0 && !(reinterpret_cast<uintptr_t>(P.G) & 7)) kloop(std::true_type{});
    else kloop(std::false_type{});
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float* row = K + row_off<!TC>(L, S.ro, i0 + u) + j0;
      if (I != J) {
        *reinterpret_cast<float4*>(row) = make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
      } else {
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (w <= u) row[w] = acc[u][w];
        if (i0 + u < n) dmax = fmaxf(dmax, fabsf(acc[u][u]));
      }
    }
  }
  }
  for (int r = tid; r < pa; r += NT) dmax = fmaxf(dmax, fabsf(e[S.act[r]]));
  float vals[1] = {dmax};
  block_reduce<NT, 0, 1>(vals, S.red);
  return vals[0];
}

// Warp-per-row dot products out[r] = Mat[r,:]·vec for r < rows (Mat global
// row-major rows×n, vec and out in shared memory); each warp keeps 4 rows in
// flight so the loads and the shuffle reductions overlap; rows of even length
// are read as float2 (one pass per row for n ≤ 64).  Not inlined: one
// copy of the code serves every call site (instruction-cache footprint).
// Ends with a barrier.
template <int NT>
__device__ __noinline__ void rowdots(const float* __restrict__ Mat, int rows, int n, const float* vec,
                                     float* out) {
  constexpr int NW = NT / 32, R = 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool v2 = !(n & 1) && !((reinterpret_cast<uintptr_t>(Mat) | reinterpret_cast<uintptr_t>(vec)) & 7);
  for (int r0 = warp * R; r0 < rows; r0 += NW * R) {
    float acc[R];
#pragma unroll
    for (int u = 0; u < R; ++u) acc[u] = 0.f;
    if (v2) {  // even n, 8-byte aligned rows: float2 loads (one pass for n ≤ 64)
      for (int j = lane; j < (n >> 1); j += 32) {
        const float2 xv = reinterpret_cast<const float2*>(vec)[j];
#pragma unroll
        for (int u = 0; u < R; ++u)
          if (r0 + u < rows) {
            const float2 g = __ldg(reinterpret_cast<const float2*>(Mat + (r0 + u) * n) + j);
            acc[u] = fmaf(g.y, xv.y, fmaf(g.x, xv.x, acc[u]));
          }
      }
    } else {
      for (int j = lane; j < n; j += 32) {
        const float xv = vec[j];
#pragma unroll
        for (int u = 0; u < R; ++u)
          if (r0 + u < rows) acc[u] = fmaf(__ldg(Mat + (r0 + u) * n + j), xv, acc[u]);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
      for (int u = 0; u < R; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
    if (lane < R && r0 + lane < rows) {
      float v = acc[0];
#pragma unroll
      for (int u = 1; u < R; ++u) v = lane == u ? acc[u] : v;
      out[r0 + lane] = v;
    }
  }
  __syncthreads();
}

// Large n (the batched engine at config-5 size: G is 8 MB per problem and
// streams from HBM): eight rows in flight per warp, float4 loads of the
// matrix and the vector; falls back to rowdots for n not a multiple of 4 or
// unaligned rows.  Ends with a barrier.
template <int NT>
__device__ __noinline__ void rowdots_large(const float* __restrict__ Mat, int rows, int n, const float* vec,
                                           float* out) {
  if ((n & 3) || ((reinterpret_cast<uintptr_t>(Mat) | reinterpret_cast<uintptr_t>(vec)) & 15)) {
    rowdots<NT>(Mat, rows, n, vec, out);
    return;
  }
  constexpr int NW = NT / 32, R = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, n4 = n >> 2;
  const float4* v4 = reinterpret_cast<const float4*>(vec);
  for (int r0 = warp * R; r0 < rows; r0 += NW * R) {
    float acc[R];
#pragma unroll
    for (int u = 0; u < R; ++u) acc[u] = 0.f;
    for (int j = lane; j < n4; j += 32) {
      const float4 xv = v4[j];
      float4 g[R];
#pragma unroll
      for (int u = 0; u < R; ++u)
        g[u] = r0 + u < rows ? __ldg(reinterpret_cast<const float4*>(Mat + (size_t)(r0 + u) * n) + j)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < R; ++u)
        acc[u] = fmaf(g[u].w, xv.w, fmaf(g[u].z, xv.z, fmaf(g[u].y, xv.y, fmaf(g[u].x, xv.x, acc[u]))));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
      for (int u = 0; u < R; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
    if (lane < R && r0 + lane < rows) {
      float v = acc[0];
#pragma unroll
      for (int u = 1; u < R; ++u) v = lane == u ? acc[u] : v;
      out[r0 + lane] = v;
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------
// Residuals (Eq. 4; Eq. 10), the norms of the relative
// stopping test (reading Q4), d₊, d₋, c, ω and the active set at (v, κ), and
// the Newton right-hand side of Eq. 14 carried to the reduced
// system:
//   f1 = −(r_t − Gᵀ(r_i + r_z − r_s)), f2 = −(r_i − r_s − c r_κ), f3 = −r_e,
//   rhs_x = f1 + Gᵀ f2 + Σ_{v_i≤0} g_i ω_i f2_i = −(r_t − Gᵀ t),
//   t_i = r_z,i + c_i r_κ + [v_i ≤ 0] ω_i f2_i;  rhs_w = f2_A;  rhs_y = f3.
// ------------------------------------------------------------------------
struct Norms {
  float gap, obj, nonfin;
  float nrt, nre, nri, nrzs, sQx, sq, sGz, sAy, sAx, sb, sGx, ss, sh, sz;
  int pa;
  bool spill;  // reading Q12c guard: the capped elimination would exceed fb_bound
};

// keep_jac (a chord step of the guarded chord relax, reading Q26): the
// Jacobian vectors d₊, d₋, c and the partition (widx, pa_keep) already in S
// are those of the cached factorisation and are kept; only the residuals are
// of the current point.  The norms do not depend on the Jacobian.
//
// pre (batched engine with Q and G shared by the batch): the GEMV products
// came from batched GEMMs over the whole batch (bnd_gemm): S.gx[0:p) = G x
// already in place, pre[0:n) = Q x, pre[n4:n4+n) = Gᵀ z; Gᵀ t is added to
// the right-hand side later (pre[2n4:], by bnd_solve), so rhs[0:n) = −r_t here.
template <int NT, bool LARGE = false>
__device__ Norms residuals(const Smem& S, const Args& a, const Prob& P, float kappa, float r_kappa,
                           bool keep_jac = false, int pa_keep = 0, const float* pre = nullptr) {
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  float mz = 0.f, ms = 0.f, mh = 0.f, mrzs = 0.f, nonfin = 0.f;
  for (int k = tid; k < p; k += NT) {
    const float zk = S.z[k], sk = S.s[k], vk = S.v[k];
    const float rz = zk - ret_b(vk, kappa), rs = sk - ret_b(-vk, kappa);
    S.rz[k] = rz; S.rs[k] = rs;
    if (!keep_jac) {
      S.c[k] = ret_dk(vk, kappa);
      S.dp[k] = ret_db(vk, kappa); S.dm[k] = ret_db(-vk, kappa);
    }
    mz = fmaxf(mz, fabsf(zk)); ms = fmaxf(ms, fabsf(sk)); mh = fmaxf(mh, fabsf(__ldg(P.h + k)));
    mrzs = fmaxf(mrzs, fmaxf(fabsf(rz), fabsf(rs)));
  }
  bool capped = false;
  int pa = pa_keep;
  if (!keep_jac) pa = compact_active<NT>(S, p, false, a.pcap, &capped);
  else __syncthreads();
  // Reading Q12c guard: when the cap bound, no eliminated constraint with
  // v_k > 0 may carry a weight ω_k = d₊/d₋ above fb_bound (every factored
  // entry stays bounded); otherwise the problem goes to the
  // uncapped fallback (block-uniform: capped is)
  bool spill = false;
  if (capped && a.fb_bound > 0.f) {
    float w = 0.f;
    for (int k = tid; k < p; k += NT)
      if (S.v[k] > 0.f && S.widx[k] < 0) w = fmaxf(w, S.dp[k] / S.dm[k]);
    float vv[1] = {w};
    block_reduce<NT, 0, 1>(vv, S.red);
    spill = vv[0] > a.fb_bound;
  }
  // rows: r_i = Gx + s − h, r_e = Ax − b (warp per row); f2, t, rhs_w, rhs_y
  if (!pre) {
    if constexpr (LARGE) rowdots_large<NT>(P.G, p, n, S.x, S.gx);
    else rowdots<NT>(P.G, p, n, S.x, S.gx);
  }
  rowdots<NT>(P.A, m, n, S.x, S.gx + p);
  for (int k = tid; k < p; k += NT) {
    const float ri = S.gx[k] + S.s[k] - __ldg(P.h + k);
    const float f2 = -(ri - S.rs[k] - S.c[k] * r_kappa);
    S.f2[k] = f2;
    const int wi = S.widx[k];
    // ω_k = d₊ for a kept constraint, d₊/d₋ for an eliminated one (Q12b, Q12c)
    const float om = wi >= 0 ? S.dp[k] : S.dp[k] / S.dm[k];
    S.om[k] = om;
    S.t[k] = fmaf(S.c[k], r_kappa, S.rz[k]) + (wi >= 0 ? 0.f : om * f2);
    if (wi >= 0) S.rhs[n4 + wi] = f2;
  }
  for (int l = tid; l < m; l += NT) S.rhs[n4 + pa + l] = -(S.gx[p + l] - __ldg(P.b + l));
  __syncthreads();
  // columns j < n: Qx, Gᵀz, Aᵀy, Gᵀt  (Q symmetric ⇒ (Qx)_j = Σ_i Q_ij x_i).
  // When n < NT the row ranges are split over ng groups of threads (partial
  // sums in S.colscr) so that every thread has work.
  const int gw = (n + 31) & ~31;
  int ng = gw >= NT ? 1 : min(NT / gw, 4), cw = gw;  // groups, column-sum stride
  // even n with 8-byte aligned rows: a thread owns the column PAIR (j, j+1)
  // (float2 loads, half the loop trips), so up to 4 groups fit for n ≤ 64;
  // used only where that gives more groups than one column per thread
  const int gw2 = ((n >> 1) + 31) & ~31;
  const int ng2 = min(min(NT, 128) / gw2, 4);
  const bool pairs = !pre && ng2 > ng && !(n & 1) &&
                     !((reinterpret_cast<uintptr_t>(P.Q) | reinterpret_cast<uintptr_t>(P.G) |
                        (m > 0 ? reinterpret_cast<uintptr_t>(P.A) : 0)) & 7);
  if (pairs) {
    ng = ng2; cw = 2 * gw2;
    const int grp = tid / gw2, jp = tid - grp * gw2, j = 2 * jp;
    if (grp < ng && j < n) {
      float2 qx = make_float2(0.f, 0.f), gz = qx, gt = qx, ay = qx;
      const int i0 = grp * n / ng, i1 = (grp + 1) * n / ng;
#pragma unroll 4
      for (int i = i0; i < i1; ++i) {
        const float2 g = __ldg(reinterpret_cast<const float2*>(P.Q + i * n + j));
        const float xi = S.x[i];
        qx.x = fmaf(g.x, xi, qx.x); qx.y = fmaf(g.y, xi, qx.y);
      }
      const int k0 = grp * p / ng, k1 = (grp + 1) * p / ng;
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const float2 g = __ldg(reinterpret_cast<const float2*>(P.G + k * n + j));
        const float zk = S.z[k], tk = S.t[k];
        gz.x = fmaf(g.x, zk, gz.x); gz.y = fmaf(g.y, zk, gz.y);
        gt.x = fmaf(g.x, tk, gt.x); gt.y = fmaf(g.y, tk, gt.y);
      }
      const int l0 = grp * m / ng, l1 = (grp + 1) * m / ng;
      for (int l = l0; l < l1; ++l) {
        const float2 g = __ldg(reinterpret_cast<const float2*>(P.A + l * n + j));
        const float yl = S.y[l];
        ay.x = fmaf(g.x, yl, ay.x); ay.y = fmaf(g.y, yl, ay.y);
      }
      float* cs = S.colscr + grp * 4 * cw;
      *reinterpret_cast<float2*>(cs + j) = qx; *reinterpret_cast<float2*>(cs + cw + j) = gz;
      *reinterpret_cast<float2*>(cs + 2 * cw + j) = gt; *reinterpret_cast<float2*>(cs + 3 * cw + j) = ay;
    }
    __syncthreads();
  } else if (ng > 1 && !pre) {
    const int grp = tid / gw, j = tid - grp * gw;
    if (grp < ng && j < n) {
      float qx = 0.f, gz = 0.f, gt = 0.f, ay = 0.f;
      const int i0 = grp * n / ng, i1 = (grp + 1) * n / ng;
#pragma unroll 4
      for (int i = i0; i < i1; ++i) qx = fmaf(__ldg(P.Q + i * n + j), S.x[i], qx);
      const int k0 = grp * p / ng, k1 = (grp + 1) * p / ng;
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const float g = __ldg(P.G + k * n + j);
        gz = fmaf(g, S.z[k], gz);
        gt = fmaf(g, S.t[k], gt);
      }
      const int l0 = grp * m / ng, l1 = (grp + 1) * m / ng;
      for (int l = l0; l < l1; ++l) ay = fmaf(__ldg(P.A + l * n + j), S.y[l], ay);
      float* cs = S.colscr + grp * 4 * gw;
      cs[j] = qx; cs[gw + j] = gz; cs[2 * gw + j] = gt; cs[3 * gw + j] = ay;
    }
    __syncthreads();
  }
  float mrt = 0.f, mqx = 0.f, mq = 0.f, mgz = 0.f, may = 0.f, obj = 0.f;
  auto col_epi = [&](int j, float qx, float gz, float gt, float ay) {
    const float qj = __ldg(P.q + j);
    const float rt = qx + qj + gz + ay;
    S.rhs[j] = -(rt - gt);
    mrt = fmaxf(mrt, fabsf(rt)); mqx = fmaxf(mqx, fabsf(qx)); mq = fmaxf(mq, fabsf(qj));
    mgz = fmaxf(mgz, fabsf(gz)); may = fmaxf(may, fabsf(ay));
    obj = fmaf(S.x[j], fmaf(0.5f, qx, qj), obj);
    if (!isfinite(rt)) nonfin += 1.f;
  };
  bool quads = false;
  if constexpr (LARGE) {
    // large n (batched engine): a thread owns a column QUAD (float4 loads of
    // Q, G, A rows) and keeps 8 rows in flight — the per-problem GEMVs of
    // config 5 (G: 8 MB per problem, from DRAM) are bound by bytes in flight
    quads = !pre && n >= 2 * NT && !(n & 3) &&
            !((reinterpret_cast<uintptr_t>(P.Q) | reinterpret_cast<uintptr_t>(P.G) |
               (m > 0 ? reinterpret_cast<uintptr_t>(P.A) : 0)) & 15);
    if (quads) {
      for (int j4 = tid; j4 < (n >> 2); j4 += NT) {
        const int j = 4 * j4;
        float4 qx = make_float4(0.f, 0.f, 0.f, 0.f), gz = qx, gt = qx, ay = qx;
        auto mat = [&](const float* M, int rows, const float* vec, const float* vec2, float4& acc, float4& acc2) {
          for (int i0 = 0; i0 < rows; i0 += 8) {
            // L2 prefetch of the rows four steps ahead, one per 128-byte line (every 8th quad)
            if (!(j4 & 7))
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (i0 + 32 + u < rows) asm volatile("prefetch.global.L2 [%0];" ::"l"(M + (size_t)(i0 + 32 + u) * n + j));
            float4 g[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              g[u] = i0 + u < rows ? __ldg(reinterpret_cast<const float4*>(M + (size_t)(i0 + u) * n + j))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (i0 + u < rows) {
                const float xv = vec[i0 + u];
                acc.x = fmaf(g[u].x, xv, acc.x); acc.y = fmaf(g[u].y, xv, acc.y);
                acc.z = fmaf(g[u].z, xv, acc.z); acc.w = fmaf(g[u].w, xv, acc.w);
                if (vec2) {
                  const float tv = vec2[i0 + u];
                  acc2.x = fmaf(g[u].x, tv, acc2.x); acc2.y = fmaf(g[u].y, tv, acc2.y);
                  acc2.z = fmaf(g[u].z, tv, acc2.z); acc2.w = fmaf(g[u].w, tv, acc2.w);
                }
              }
            }
          }
        };
        float4 dummy;
        mat(P.Q, n, S.x, nullptr, qx, dummy);
        mat(P.G, p, S.z, S.t, gz, gt);
        mat(P.A, m, S.y, nullptr, ay, dummy);
        col_epi(j, qx.x, gz.x, gt.x, ay.x);
        col_epi(j + 1, qx.y, gz.y, gt.y, ay.y);
        col_epi(j + 2, qx.z, gz.z, gt.z, ay.z);
        col_epi(j + 3, qx.w, gz.w, gt.w, ay.w);
      }
    }
  }
  for (int j = tid; !quads && j < n; j += NT) {
    float qx = 0.f, gz = 0.f, gt = 0.f, ay = 0.f;
    if (pre) {  // Q x and Gᵀ z from the batched GEMMs; Gᵀ t added by bnd_solve
      qx = pre[j];
      gz = pre[a.n4 + j];
      for (int l = 0; l < m; ++l) ay = fmaf(__ldg(P.A + l * n + j), S.y[l], ay);
    } else if (ng > 1) {
      for (int g = 0; g < ng; ++g) {
        const float* cs = S.colscr + g * 4 * cw;
        qx += cs[j]; gz += cs[cw + j]; gt += cs[2 * cw + j]; ay += cs[3 * cw + j];
      }
    } else {
#pragma unroll 4
      for (int i = 0; i < n; ++i) qx = fmaf(__ldg(P.Q + i * n + j), S.x[i], qx);
#pragma unroll 4
      for (int k = 0; k < p; ++k) {
        const float g = __ldg(P.G + k * n + j);
        gz = fmaf(g, S.z[k], gz);
        gt = fmaf(g, S.t[k], gt);
      }
      for (int l = 0; l < m; ++l) ay = fmaf(__ldg(P.A + l * n + j), S.y[l], ay);
    }
    col_epi(j, qx, gz, gt, ay);
  }
  for (int j = n + tid; j < n4; j += NT) S.rhs[j] = 0.f;
  const int N = n4 + pa + m;
  for (int j = N + tid; j < r4(N); j += NT) S.rhs[j] = 0.f;
  float mri = 0.f, mgx = 0.f, mre = 0.f, max_ = 0.f, mb = 0.f, gap = 0.f;
  for (int k = tid; k < p; k += NT) {
    const float gx = S.gx[k];
    const float ri = gx + S.s[k] - __ldg(P.h + k);
    if (!isfinite(ri)) nonfin += 1.f;
    mri = fmaxf(mri, fabsf(ri)); mgx = fmaxf(mgx, fabsf(gx));
    gap = fmaf(S.s[k], S.z[k], gap);
  }
  for (int l = tid; l < m; l += NT) {
    const float ax = S.gx[p + l], bl = __ldg(P.b + l);
    mre = fmaxf(mre, fabsf(ax - bl)); max_ = fmaxf(max_, fabsf(ax)); mb = fmaxf(mb, fabsf(bl));
  }
  float v[17] = {gap, obj, nonfin, mrt, mre, mri, mrzs, mqx, mq, mgz, may, max_, mb, mgx, ms, mh, mz};
  block_reduce<NT, 3, 14>(v, S.red);
  Norms R;
  R.gap = v[0]; R.obj = v[1]; R.nonfin = v[2]; R.nrt = v[3]; R.nre = v[4]; R.nri = v[5]; R.nrzs = v[6];
  R.sQx = v[7]; R.sq = v[8]; R.sGz = v[9]; R.sAy = v[10]; R.sAx = v[11]; R.sb = v[12]; R.sGx = v[13];
  R.ss = v[14]; R.sh = v[15]; R.sz = v[16];
  R.pa = pa;
  R.spill = spill;
  return R;
}

__device__ __forceinline__ bool feasible_rel(const Norms& R, float tol) {
  const float st = fmaxf(1.f, fmaxf(fmaxf(R.sQx, R.sq), fmaxf(R.sGz, R.sAy)));
  const float se = fmaxf(1.f, fmaxf(R.sAx, R.sb));
  const float si = fmaxf(1.f, fmaxf(R.sGx, fmaxf(R.ss, R.sh)));
  const float sz = fmaxf(1.f, fmaxf(R.sz, R.ss));
  return R.nrt <= tol * st && R.nre <= tol * se && R.nri <= tol * si && R.nrzs <= tol * sz;
}
// phi = largest of the four relative residuals (feasible_rel <=> phi <= tol).
__device__ __forceinline__ float rel_phi(const Norms& R) {
  const float st = fmaxf(1.f, fmaxf(fmaxf(R.sQx, R.sq), fmaxf(R.sGz, R.sAy)));
  const float se = fmaxf(1.f, fmaxf(R.sAx, R.sb));
  const float si = fmaxf(1.f, fmaxf(R.sGx, fmaxf(R.ss, R.sh)));
  const float sz = fmaxf(1.f, fmaxf(R.sz, R.ss));
  return fmaxf(fmaxf(R.nrt / st, R.nre / se), fmaxf(R.nri / si, R.nrzs / sz));
}
// Reading Q5b: Alg. 2 stops (with κ at κ_relax) when phi <= relax_tol, or
// phi <= tol and the last Newton step did not reduce phi by 10% (f32 floor).
__device__ __forceinline__ bool relax_done(const Norms& R, float tol, float relax_tol, float phi_prev) {
  const float phi = rel_phi(R);
  return phi <= relax_tol || (phi <= tol && phi > 0.9f * phi_prev);
}
__device__ __forceinline__ bool converged_solve(const Norms& R, float tol) {
  return feasible_rel(R, tol) && R.gap <= tol * fmaxf(1.f, fabsf(R.obj));
}

// v = z − s and κ = sᵀz/p (Alg. 1 lines 5-6; divisor p: reading Q1)
template <int NT>
__device__ float manifold_coords(const Smem& S, const Args& a) {
  float gap = 0.f;
  for (int k = threadIdx.x; k < a.p; k += NT) {
    S.v[k] = S.z[k] - S.s[k];
    gap = fmaf(S.s[k], S.z[k], gap);
  }
  float v[1] = {gap};
  block_reduce<NT, 1, 0>(v, S.red);
  return a.p > 0 ? v[0] / (float)a.p : 0.f;
}

// Recover Δv from the reduced solution: Δv_i = g_iᵀΔx + w_i with w_i solved
// (i ∈ A) or eliminated: w_i = (d₊_i g_iᵀΔx − f2_i)/d₋_i (v_i ≤ 0).  Writes
// S.gx[k] = Δv_k.  (f2 = 0 for the adjoint.)
template <int NT, bool LARGE = false>
__device__ void recover_dv(const Smem& S, const Args& a, const Prob& P, bool zero_f2, bool gx_ready = false) {
  const int n4 = a.n4;
  if (!gx_ready) {  // (gx_ready: G Δx from a batched GEMM)
    if constexpr (LARGE) rowdots_large<NT>(P.G, a.p, a.n, S.rhs, S.gx);
    else rowdots<NT>(P.G, a.p, a.n, S.rhs, S.gx);
  }
  for (int k = threadIdx.x; k < a.p; k += NT) {
    const float gdx = S.gx[k];
    const int wi = S.widx[k];
    const float w = wi >= 0 ? S.rhs[n4 + wi] : (S.dp[k] * gdx - (zero_f2 ? 0.f : S.f2[k])) / S.dm[k];
    S.gx[k] = gdx + w;
  }
  __syncthreads();
}

// Δκ = −r_κ; Δz = −r_z + d₊Δv + cΔκ; Δs = −r_s − d₋Δv + cΔκ (Eq. 13 rows
// 4-6); α = min(1, τ α_max) (Eq. 6 + Q3); step on (x, y, v, κ) and retract
// (P:425-429).  Returns false (iterate untouched) if the direction is not
// finite.
template <int NT, bool LARGE = false>
__device__ bool newton_update(const Smem& S, const Args& a, const Prob& P, int pa, float& kappa, float r_kappa,
                              int* stage, bool gx_ready = false) {
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  const float dk = -r_kappa;
  recover_dv<NT, LARGE>(S, a, P, false, gx_ready);
  float amax = INFINITY, bad = 0.f;
  for (int k = tid; k < p; k += NT) {
    const float dv = S.gx[k];
    const float dz = -S.rz[k] + S.dp[k] * dv + S.c[k] * dk;
    const float ds = -S.rs[k] - S.dm[k] * dv + S.c[k] * dk;
    if (ds < 0.f) amax = fminf(amax, -S.s[k] / ds);
    if (dz < 0.f) amax = fminf(amax, -S.z[k] / dz);
    if (!isfinite(dz) || !isfinite(ds)) bad = 1.f;
  }
  for (int j = tid; j < n; j += NT) if (!isfinite(S.rhs[j])) bad = 1.f;
  for (int l = tid; l < m; l += NT) if (!isfinite(S.rhs[n4 + pa + l])) bad = 1.f;
  float vals[1] = {bad};
  block_reduce<NT, 0, 1>(vals, S.red);
  const float am = block_min<NT>(amax, S.red + 64);
  if (vals[0] > 0.f) { *stage = STG_CORRECTOR; return false; }
  const float alpha = fminf(1.f, a.tau * am);
  if (!(alpha > 0.f)) { *stage = STG_LINESEARCH; return false; }
  for (int j = tid; j < n; j += NT) S.x[j] = fmaf(alpha, S.rhs[j], S.x[j]);
  for (int l = tid; l < m; l += NT) S.y[l] = fmaf(alpha, S.rhs[n4 + pa + l], S.y[l]);
  const float kn = fmaf(alpha, dk, kappa);
  for (int k = tid; k < p; k += NT) {
    const float vn = fmaf(alpha, S.gx[k], S.v[k]);
    S.z[k] = ret_b(vn, kn);
    S.s[k] = ret_b(-vn, kn);
  }
  kappa = kn;
  __syncthreads();
  return true;
}

// Alg. 3 parameter gradients from (x, y, z) and (dx, dy, dz) in
// shared memory; coalesced stores; per-problem vectors for shared-field sums.
template <int NT>
__device__ void write_gradients(const Smem& S, const Args& a, const int bid) {
  const int tid = threadIdx.x;
  const int n = a.n, p = a.p, m = a.m;
  const long long bb = bid;
  // (row, column) of element e = tid + s·NT advanced without a division
  const int drr = NT / n, dj = NT - drr * n, r0 = tid / n, j0 = tid - r0 * n;
  auto adv = [&](int& r, int& j) { r += drr; j += dj; if (j >= n) { j -= n; ++r; } };
  if (a.gQ) {
    float* o = a.gQ + bb * n * n;
    int i = r0, j = j0;
    for (int e = tid; e < n * n; e += NT, adv(i, j)) o[e] = 0.5f * (S.dx[i] * S.x[j] + S.x[i] * S.dx[j]);
  }
  if (a.gq) for (int j = tid; j < n; j += NT) a.gq[bb * n + j] = S.dx[j];
  if (a.gA) {
    float* o = a.gA + bb * m * n;
    int l = r0, j = j0;
    for (int e = tid; e < m * n; e += NT, adv(l, j)) o[e] = S.dy[l] * S.x[j] + S.y[l] * S.dx[j];
  }
  if (a.gb) for (int l = tid; l < m; l += NT) a.gb[bb * m + l] = -S.dy[l];
  if (a.gG) {
    float* o = a.gG + bb * p * n;
    int i = r0, j = j0;
    for (int e = tid; e < p * n; e += NT, adv(i, j)) o[e] = S.dz[i] * S.x[j] + S.z[i] * S.dx[j];
  }
  if (a.gh) for (int i = tid; i < p; i += NT) a.gh[bb * p + i] = -S.dz[i];
  if (a.wx) {
    for (int j = tid; j < n; j += NT) { a.wx[bb * n + j] = S.x[j]; a.wdx[bb * n + j] = S.dx[j]; }
    for (int l = tid; l < m; l += NT) { a.wy[bb * m + l] = S.y[l]; a.wdy[bb * m + l] = S.dy[l]; }
    for (int i = tid; i < p; i += NT) { a.wz[bb * p + i] = S.z[i]; a.wdz[bb * p + i] = S.dz[i]; }
  }
}

// ------------------------------------------------------------------------
// One problem, either direction, in ONE Newton loop (so that the solve and
// the backward launches run the same code: they share the instruction cache
// when the backward grid overlaps the end of the solve grid).
//   solve (bwd = false): CVXOPT initialisation (Q11; iteration −1) +
//     Algorithm 1: κ_target = σκ, stop on the relative test (Q4).
//   backward (bwd = true): Algorithm 2 (Q5, Q5b, Q6) from the
//     solution: κ_target = κ_relax, Newton steps until the relax test holds;
//     at that point the KKT matrix is assembled and factored once more at the
//     relaxed point and Algorithm 3 (Q7, Q8) solves it with the
//     right-hand side (−∇ₓℓ, 0, 0) — the factorisation Alg. 3 reuses sits
//     at the relaxed point, as in factor-then-check (Q6).
// assemble / factor / solve_qd have ONE call site.
// ------------------------------------------------------------------------
template <int NT, bool BIG, int MAXN4 = 256>
__device__ __forceinline__ void ipm_problem(const Args& a, const Smem& S, const int bid, const bool bwd,
                                            const bool lost = false) {
  const int tid = threadIdx.x;
  const Prob P = prob_of(a, bid);
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  int status = ST_CONVERGED, it = 0;
  bool ok = false;  // backward: gradients computed
  float fl = 0.f;   // algorithmic flops of this problem
  float phi_prev = INFINITY;
  unsigned long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64();
  bool handed = false;  // reading Q12c guard: this problem goes to the fallback launch
  // guarded chord relax (reading Q26; path 1 only).  Solve: cached = this
  // problem stored the factorisation of its first iterate with κ < √10·κ_relax
  // (chord cache of Args).  Backward: chord = chord steps on it are being taken.
  const bool chord_on = !BIG && a.kc && a.relax_mode == 2;
  bool cached = false, chord = false;
  int nchord = 0;
  float psi_prev = INFINITY;
  if (chord_on && !bwd && tid == 0) a.chord_ok[bid] = 0;
  if (a.fb_bound > 0.f) {
    if (!bwd) {
      if (tid == 0) a.fb_flag[bid] = 0;
    } else if (__ldcg(a.fb_flag + bid)) {  // the solve handed it over: so does the backward
      if (tid == 0) a.fb_list[atomicAdd(a.fb_count, 1)] = bid;
      return;
    }
  }
  if (bwd) {
    // the solve's outputs (written by other SMs in this or the previous
    // kernel): read past L1
    for (int j = tid; j < n; j += NT) S.x[j] = __ldcg(a.x + (long long)bid * n + j);
    for (int l = tid; l < m; l += NT) S.y[l] = __ldcg(a.y + (long long)bid * m + l);
    for (int i = tid; i < p; i += NT) {
      S.z[i] = __ldcg(a.z + (long long)bid * p + i);
      S.s[i] = __ldcg(a.s + (long long)bid * p + i);
    }
    __syncthreads();
    if (lost) status = ST_FAIL | (STG_BACKWARD << 8);
    else if ((__ldcg(a.status + bid) & 0xff) != ST_CONVERGED) status = ST_FAIL | (STG_RELAX << 8);
    chord = chord_on && __ldcg(a.chord_ok + bid) != 0;
  }
  for (int k = bwd ? 0 : -1; status == ST_CONVERGED; ++k) {
    const bool init = k < 0;
    float kappa = 0.f, kt = 0.f;
    int pa = 0;
    bool adj = false;  // backward: relaxed — this iteration's solve is Alg. 3's
    bool chord_step = false;  // backward: a chord step on the solve's cached factorisation (Q26)
    bool cache = false;       // solve: this iteration's factorisation goes to the chord cache
    const float *cw = S.om, *ev = S.om;
    if (init) {
      // [[Q, Gᵀ, Aᵀ], [G, −I, 0], [A, 0, 0]] (x, ẑ, y) = (−q, h, b); the congruence
      // ẑ = Gx + w decouples w = −h: reduced matrix [[Q + GᵀG, Aᵀ], [A, 0]],
      // right-hand side (−q + Gᵀh, b); ẑ = Gx − h.
      for (int i = tid; i < p; i += NT) { S.om[i] = 1.f; S.v[i] = -1.f; }
      __syncthreads();
      compact_active<NT>(S, p, true, p);
      for (int j = tid; j < n4; j += NT) {
        float acc = 0.f;
        if (j < n) {
          acc = -__ldg(P.q + j);
          for (int i = 0; i < p; ++i) acc = fmaf(__ldg(P.G + i * n + j), __ldg(P.h + i), acc);
        }
        S.rhs[j] = acc;
      }
      for (int l = tid; l < m; l += NT) S.rhs[n4 + l] = __ldg(P.b + l);
      for (int j = n4 + m + tid; j < r4(n4 + m); j += NT) S.rhs[j] = 0.f;
    } else {
      kappa = manifold_coords<NT>(S, a);
      kt = bwd ? a.kappa_relax : a.sigma * kappa;  // κ_target: κ_relax (Alg. 2) or σκ (Alg. 1)
      const float* cj = chord_on ? a.chd + (long long)bid * a.chd_stride : nullptr;
      const bool was_chord = chord;
      if (was_chord) {  // the cached Jacobian: the right-hand side of a chord step
        const int p4 = (p + 3) & ~3;
        for (int i = tid; i < p; i += NT) {
          S.dp[i] = __ldcg(cj + 4 + i); S.dm[i] = __ldcg(cj + 4 + p4 + i); S.c[i] = __ldcg(cj + 4 + 2 * p4 + i);
          S.widx[i] = __float_as_int(__ldcg(cj + 4 + 3 * p4 + i));
        }
        __syncthreads();
      }
      // one call site; a second pass (current Jacobian) when a chord phase ends
      bool keep = was_chord, fin = false;
      Norms R;
#pragma unroll 1
      for (int pass = 0;; ++pass) {
        R = residuals<NT>(S, a, P, kappa, kappa - kt, keep, keep ? __float_as_int(__ldcg(cj)) : 0);
        if (pass == 1 || !was_chord || R.spill || R.nonfin > 0.f) break;
        const bool kok = p == 0 || fabsf(kappa / a.kappa_relax - 1.f) <= a.relax_ktol;
        const float psi = fmaxf(rel_phi(R), p == 0 ? 0.f : fabsf(kappa / a.kappa_relax - 1.f));
        if (nchord >= a.chord_max || (nchord > 0 && !(psi <= a.chord_rho * psi_prev))) {
          chord = false;
          phi_prev = INFINITY;  // the stall test (Q5b) measures Newton steps only
        }
        psi_prev = psi;
        // a chord stops only at φ ≤ relax_tol (a slow chord is not the f32 floor)
        adj = kok && (chord ? rel_phi(R) <= a.relax_tol : relax_done(R, a.tol, a.relax_tol, phi_prev));
        fin = !adj && k == a.relax_max_iter;
        if (fin || !(adj || !chord)) break;
        chord = false;
        keep = false;
        __syncthreads();
      }
      long long t1 = clock64(); tph[0] += t1 - t0; t0 = t1;
      it = k;
      if (R.spill) {
        handed = true;
        status = ST_FAIL;  // (placeholder: the fallback launch overwrites this problem's outputs)
        if (tid == 0) {
          if (!bwd) a.fb_flag[bid] = 1;
          a.fb_list[atomicAdd(a.fb_count, 1)] = bid;
        }
        break;
      }
      if (R.nonfin > 0.f) { status = ST_FAIL | ((bwd ? STG_RELAX : STG_SCALING) << 8); break; }
      if (!bwd) {
        fl += iter_flops(n, m, p, 0, true, false, false);
        if (converged_solve(R, a.tol)) break;
        if (k == a.max_iter) { status = ST_MAX_ITER; break; }
        fl -= iter_flops(n, m, p, 0, true, false, false);  // counted again below with the step
        if (chord_on && !cached && kappa < sqrtf(10.f) * a.kappa_relax) cache = cached = true;
      } else {
        const bool kok = p == 0 || fabsf(kappa / a.kappa_relax - 1.f) <= a.relax_ktol;
        if (!was_chord) adj = kok && relax_done(R, a.tol, a.relax_tol, phi_prev);
        phi_prev = kok ? rel_phi(R) : INFINITY;
        if (!adj && k == a.relax_max_iter) { status = ST_MAX_ITER | (STG_RELAX << 8); break; }
        chord_step = chord;
        if (chord_step) ++nchord;
      }
      pa = R.pa;
      cw = S.dp; ev = S.dm;
    }
    const KLayout L = KLayout::make(n4 + pa + m, n4);
    float* const K = kkt_ptr<BIG>(S, a, L);
    tph[5] += pa; tph[6] += L.N; tph[7] = tph[7] > (unsigned long long)L.N ? tph[7] : (unsigned long long)L.N;
    long long t1;
    if (chord_step) {
      // the solve's cached factorisation (reading Q26) into the KKT buffer
      fl += iter_flops(n, m, p, pa, true, false, true);
      const float4* src = reinterpret_cast<const float4*>(a.kc + (long long)bid * a.kc_stride);
      float4* dst = reinterpret_cast<float4*>(K);
      for (int i = tid; i < (L.size() + 3) >> 2; i += NT) dst[i] = __ldcg(src + i);
      const float* cr = a.chd + (long long)bid * a.chd_stride + 4 + 4 * ((p + 3) & ~3);
      for (int i = tid; i < L.N4; i += NT) S.rinv[i] = __ldcg(cr + i);
      if constexpr (!BIG) for (int i = tid; i < L.N4; i += NT) S.ro[i] = L.off(i);
      __syncthreads();
      t1 = clock64(); tph[2] += t1 - t0; t0 = t1;
    } else {
      fl += iter_flops(n, m, p, pa, !init, true, true);
      const float dmax = assemble<NT, BIG>(K, S, a, P, L, pa, S.om, cw, ev);
      t1 = clock64(); tph[1] += t1 - t0; t0 = t1;
      factor_any<NT, BIG, MAXN4>(K, S, L, a.floor_rel * dmax);
      t1 = clock64(); tph[2] += t1 - t0; t0 = t1;
      if (cache) {  // Alg. 1's factorisation nearest κ_relax: to the chord cache (reading Q26)
        float4* dst = reinterpret_cast<float4*>(a.kc + (long long)bid * a.kc_stride);
        const float4* src = reinterpret_cast<const float4*>(K);
        for (int i = tid; i < (L.size() + 3) >> 2; i += NT) dst[i] = src[i];
        float* cj = a.chd + (long long)bid * a.chd_stride;
        const int p4 = (p + 3) & ~3;
        for (int i = tid; i < p; i += NT) {
          cj[4 + i] = S.dp[i]; cj[4 + p4 + i] = S.dm[i]; cj[4 + 2 * p4 + i] = S.c[i];
          cj[4 + 3 * p4 + i] = __int_as_float(S.widx[i]);
        }
        for (int i = tid; i < L.N4; i += NT) cj[4 + 4 * p4 + i] = S.rinv[i];
        if (tid == 0) {
          cj[0] = __int_as_float(pa); cj[1] = kappa;
          a.chord_ok[bid] = 1;
        }
      }
    }
    if (adj) {
      // Algorithm 3: reduced system with right-hand side (−∇ₓℓ, 0, 0).  The
      // cotangent may be the output of the kernel launched just before this
      // one on the stream (programmatic launch: this grid may have started
      // while that one still runs), so wait for it to complete first; the
      // relax steps above read only this ctx's solve outputs (done[] flags).
      grid_dependency_wait();
      for (int j = tid; j < L.N4; j += NT) S.rhs[j] = j < n ? -__ldg(a.dl + (long long)bid * n + j) : 0.f;
      __syncthreads();
    }
    if constexpr (BIG) solve_qd<NT>(K, L, S.rinv, S.rhs);
    else solve_qd<NT, true>(K, L, S.rinv, S.rhs, S.ro);
    t1 = clock64(); tph[3] += t1 - t0; t0 = t1;
    if (init) {
      for (int j = tid; j < n; j += NT) S.x[j] = S.rhs[j];
      for (int l = tid; l < m; l += NT) S.y[l] = S.rhs[n4 + l];
      __syncthreads();
      rowdots<NT>(P.G, p, n, S.x, S.dz);
      for (int i = tid; i < p; i += NT) S.dz[i] -= __ldg(P.h + i);  // ẑ = Gx − h
      float ap = -INFINITY, ad = -INFINITY, bad = 0.f;
      for (int i = tid; i < p; i += NT) {
        const float zh = S.dz[i];
        ap = fmaxf(ap, zh); ad = fmaxf(ad, -zh);
        if (!isfinite(zh)) bad = 1.f;
      }
      for (int j = tid; j < n; j += NT) if (!isfinite(S.x[j])) bad = 1.f;
      float v[3] = {ap, ad, bad};
      block_reduce<NT, 0, 3>(v, S.red);
      ap = v[0]; ad = v[1];
      for (int i = tid; i < p; i += NT) {  // s~ = −ẑ, z~ = ẑ, shifted into the interior
        const float zh = S.dz[i];
        S.s[i] = ap >= 0.f ? -zh + (1.f + ap) : -zh;
        S.z[i] = ad >= 0.f ? zh + (1.f + ad) : zh;
      }
      __syncthreads();
      if (v[2] > 0.f) { status = ST_FAIL | (STG_INIT << 8); break; }
    } else if (adj) {
      // dv = G dx + w (w eliminated for v_i ≤ 0 with f2 = 0), dz = d₊ ⊙ dv
      recover_dv<NT>(S, a, P, true);
      for (int i = tid; i < p; i += NT) S.dz[i] = S.dp[i] * S.gx[i];
      for (int j = tid; j < n; j += NT) S.dx[j] = S.rhs[j];
      for (int l = tid; l < m; l += NT) S.dy[l] = S.rhs[n4 + pa + l];
      __syncthreads();
      float bad = 0.f;
      for (int j = tid; j < n; j += NT) if (!isfinite(S.dx[j])) bad = 1.f;
      for (int i = tid; i < p; i += NT) if (!isfinite(S.dz[i])) bad = 1.f;
      for (int l = tid; l < m; l += NT) if (!isfinite(S.dy[l])) bad = 1.f;
      float v[1] = {bad};
      block_reduce<NT, 0, 1>(v, S.red);
      ok = !(v[0] > 0.f);
      if (!ok) status = ST_FAIL | (STG_BACKWARD << 8);
      break;
    } else {
      int stage = 0;
      if (!newton_update<NT>(S, a, P, pa, kappa, kappa - kt, &stage)) {
        status = ST_FAIL | ((bwd ? STG_RELAX : stage) << 8);
        break;
      }
    }
    t1 = clock64(); tph[4] += t1 - t0; t0 = t1;
  }
  if (!bwd) {
    if (a.prof && tid == 0)
      for (int i = 0; i < 8; ++i) a.prof[bid * 8 + i] = tph[i];
    for (int j = tid; j < n; j += NT) a.x[(long long)bid * n + j] = S.x[j];
    for (int l = tid; l < m; l += NT) a.y[(long long)bid * m + l] = S.y[l];
    for (int i = tid; i < p; i += NT) {
      a.z[(long long)bid * p + i] = S.z[i];
      a.s[(long long)bid * p + i] = S.s[i];
    }
    if (tid == 0) {
      a.iters[bid] = it;
      a.status[bid] = status;
      if (a.status_out) a.status_out[bid] = status;
      if (a.flops) a.flops[bid] = fl;
    }
  } else {
    if (handed) {  // the fallback launch writes this problem's gradients
      __syncthreads();
      return;
    }
    // the gradient buffers may still be read by the previous kernel on the
    // stream (caching allocator reuse): no store before it has completed
    grid_dependency_wait();
    if (!ok) {  // zero-filled gradients for failed problems
      for (int j = tid; j < n; j += NT) { S.dx[j] = 0.f; S.x[j] = 0.f; }
      for (int l = tid; l < m; l += NT) { S.dy[l] = 0.f; S.y[l] = 0.f; }
      for (int i = tid; i < p; i += NT) { S.dz[i] = 0.f; S.z[i] = 0.f; }
      __syncthreads();
    }
    write_gradients<NT>(S, a, bid);
    if (tid == 0) {
      if (nchord > 0 && a.chord_cnt) atomicAdd(a.chord_cnt, nchord);
      if (a.riters) a.riters[bid] = it;
      if (a.rstatus) a.rstatus[bid] = status;
      if (a.flops) a.flops[bid] = fl + 2.f * (n * n + m * n + p * n);  // + gradient outer products
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------
// The kernel: persistent CTAs, problems handed out by next_problem.
// NT = 128 (path 1 at 3-4 CTAs/SM, reduced systems ≤ MAXN4 = 256 rows),
// NT = 256 (path 1 at 1-2 CTAs/SM, and the large-N kernels), NT = 64 (small-n path: two warps own one QP, systems ≤ 64 rows,
// up to 8 problems per SM).
// a.bwd = 0: solve launch (qp_solve_batched); each finished problem is
//   published in done[b] = epoch (release).
// a.bwd = 1: backward launch (qp_backward_batched), possibly started while
//   the solve grid drains (programmatic stream serialisation): each problem
//   first waits for done[b] == epoch.
// ------------------------------------------------------------------------
template <int NT, int MINB, bool BIG, int MAXN4 = 256>
__global__ void __launch_bounds__(NT, MINB) ipm_kernel(const Args a) {
  extern __shared__ __align__(16) float smem[];
  const Smem S = carve(smem, a);
  const bool bwd = a.bwd != 0;
  // lets the next launch on the stream (the backward) start on SMs this grid leaves idle
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if constexpr (BIG) tc::tmem_alloc(tc::tc_state(S.tc));
  for (int bid = next_problem(a, S.flag + 12); bid < a.B; bid = next_problem(a, S.flag + 12)) {
    bool lost = false;  // backward: the solve never published this problem (watchdog)
    if (bwd && a.done) {
      if (threadIdx.x == 0) {
        // relaxed polling (an acquire per poll would invalidate this SM's L1),
        // one acquire fence once the flag is seen; after 20 s without the
        // flag the problem is reported failed instead of hanging the GPU
        int e;
        const unsigned long long t0 = gtimer();
        for (;;) {
          asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(e) : "l"(a.done + bid) : "memory");
          if (e == a.epoch) break;
          if (gtimer() - t0 > 20000000000ull) { lost = true; break; }
          __nanosleep(256);
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      lost = __syncthreads_or(lost);
    }
    if (a.tl && threadIdx.x == 0) { a.tl[3 * bid] = smid(); a.tl[3 * bid + 1] = gtimer(); }
    ipm_problem<NT, BIG, MAXN4>(a, S, bid, bwd, lost);  // ends with a barrier after the output stores
    if (a.tl && threadIdx.x == 0) a.tl[3 * bid + 2] = gtimer();
    if (!bwd && a.done && threadIdx.x == 0)  // release (cumulative through the barrier): outputs before the flag
      asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(a.done + bid), "r"(a.epoch) : "memory");
  }
  // a programmatically launched backward completes only after the grid it
  // depends on (so that work ordered after it, e.g. the fallback launch,
  // also follows that grid)
  if (bwd) grid_dependency_wait();
  if constexpr (BIG) tc::tmem_free(*tc::tc_state(S.tc).tmem_slot);
}

// ------------------------------------------------------------------------
// Batch sums for shared parameters (K8 of SURVEY §2.4; Alg. 3 formulas summed
// over the batch):  out[r][c] = scale · Σ_b (U[b][r] V[b][c] + U2[b][r] V2[b][c])
// 64×64 output tile per CTA, 256 threads, 4×4 outputs per thread; the batch
// dimension is staged through shared memory 32 rows at a time.
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256) outer_sum_kernel(const float* __restrict__ U, const float* __restrict__ V,
                                                        const float* __restrict__ U2, const float* __restrict__ V2,
                                                        int B, int R, int Cc, float scale, float* __restrict__ out) {
  __shared__ float su[2][32][64], sv[2][32][64];
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  float acc[4][4] = {};
  for (int b0 = 0; b0 < B; b0 += 32) {
    for (int e = tid; e < 32 * 64; e += 256) {
      const int bb = e >> 6, k = e & 63;
      const int b = b0 + bb;
      const bool okb = b < B;
      su[0][bb][k] = (okb && r0 + k < R) ? U[(long long)b * R + r0 + k] : 0.f;
      sv[0][bb][k] = (okb && c0 + k < Cc) ? V[(long long)b * Cc + c0 + k] : 0.f;
      su[1][bb][k] = (okb && r0 + k < R) ? U2[(long long)b * R + r0 + k] : 0.f;
      sv[1][bb][k] = (okb && c0 + k < Cc) ? V2[(long long)b * Cc + c0 + k] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int bb = 0; bb < 32; ++bb) {
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        float u[4], v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { u[i] = su[w][bb][tr + 16 * i]; v[i] = sv[w][bb][tc + 16 * i]; }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(u[i], v[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + tr + 16 * i, c = c0 + tc + 16 * j;
      if (r < R && c < Cc) out[(long long)r * Cc + c] = scale * acc[i][j];
    }
}

// out[c] = scale · Σ_b U[b][c]
__global__ void __launch_bounds__(256) col_sum_kernel(const float* __restrict__ U, int B, int Cc, float scale,
                                                      float* __restrict__ out) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= Cc) return;
  float acc = 0.f;
  for (int b = 0; b < B; ++b) acc += U[(long long)b * Cc + c];
  out[c] = scale * acc;
}

}  // namespace qpb
