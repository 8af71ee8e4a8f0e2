// qpb200.cu — host side of the C ABI declared in include/qpb200.h: context,
// validation, workspace management, dispatch and stream-ordered launches.
// Every step of the hot path runs in the kernels of ipm_kernels.cuh; this file
// only marshals.  There is no CPU fallback: without a CUDA device every entry
// point returns QP_ERR_CUDA.
#include <cuda.h>  // CUtensorMap (types only: the encoder comes from cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <new>

#include <algorithm>
#include <vector>

#include "../../include/qpb200.h"
#include "xpm_kernels.cuh"
#include "tc_syrk.cuh"
#include "bnd_kernels.cuh"

namespace {

// Two kernel shapes: path 1 (the whole KKT system in shared memory, 128
// threads, 1-4 CTAs/SM) and the large-N kernels (256 threads, 1 CTA/SM,
// tensor-core assembly, KKT system in smem or in a per-CTA global workspace).
constexpr size_t kMaxSmem = 232448;  // 227 KB opt-in dynamic shared memory per CTA (sm_100a)

struct Layout {
  int n4, Nmax, N4max;
  int ksmem, ncap;       // shared-memory KKT buffer and the largest reduced system it holds
  int pcap;              // path 1: largest kept set |A| (reading Q12c; p = no cap)
  long long kglob;       // global workspace floats per CTA (worst case)
  bool big;              // some reduced systems may exceed 256 rows (factor_big compiled in)
  bool batched;          // big shapes: the batched phase engine (bnd_kernels.cuh, path 4)
  int threads, minb;     // kernel shape
  size_t smem;
};

// floats of the tcgen05 staging area the large-N kernels carry
int tc_floats(bool big) { return big ? qpb::tc::SMEM_BYTES / 4 : 0; }

// entries of the shared-memory row-offset table (path 1 kernels only)
int ro_ints(const Layout& L, bool big) { return big ? 0 : L.N4max; }

// path 1 at buffer capacity ncap (the vectors sized for ncap as well)
size_t path1_smem(const Layout& L, int m, int p, int ncap) {
  const int N4 = (ncap + 3) & ~3;
  return qpb::ipm_smem_bytes(L.n4, m, p, N4, qpb::KLayout::make(ncap, L.n4).size(), 0, N4);
}

size_t smem_for(const Layout& L, int m, int p, int ncap, bool big) {
  const int ks = ncap > 0 ? qpb::KLayout::make(ncap, L.n4).size() : 0;
  return qpb::ipm_smem_bytes(L.n4, m, p, L.N4max, ks, tc_floats(big), ro_ints(L, big));
}

// Shared-memory budget per CTA (dynamic part) for `ctas` CTAs per SM.
size_t budget(int ctas) { return std::min(kMaxSmem, (size_t)(233472 / ctas) - 1024); }

Layout make_layout(int n, int m, int p, int formulation, int batch = 0, int sms = 148, bool force_big = false) {
  Layout L;
  L.n4 = (n + 3) & ~3;
  // implicit: reduced system n4 + |A| + m with |A| <= p; standard arm: every
  // constraint condensed into H = Q + GᵀD(z/s)G, so n4 + m
  L.Nmax = L.n4 + (formulation == QP_EXPLICIT ? 0 : p) + m;
  L.N4max = (L.Nmax + 3) & ~3;
  L.kglob = qpb::KLayout::make(L.Nmax, L.n4).size();
  L.big = false;
  L.batched = false;
  // Path 1 (below) when the worst case has at most 256 rows and a buffer of
  // the size it needs fits; otherwise the large-N kernels: one CTA per SM
  // with the largest smem buffer, iterations with a larger reduced system in
  // the CTA's global workspace (hybrid).
  int env_cap = -1;
  if (const char* e = getenv("QPB200_NCAP")) env_cap = atoi(e);
  int env_ctas = 0;
  if (const char* e = getenv("QPB200_CTAS")) env_ctas = atoi(e);
  L.threads = 128; L.minb = 1; L.ncap = 0; L.pcap = p;
  // path 1: the KKT buffer and the register-panel factorisation (N4 ≤ 256).
  // Take the largest CTA count (≤ 4) whose buffer holds either the worst case
  // n4 + p + m or, with the kept set capped (reading Q12c), at least
  // n4 + min(p, n4) + m rows: room for every constraint that can be strongly
  // active at a solution satisfying LICQ (at most n of them), so the cap only
  // ever eliminates constraints far from active.  More co-resident problems
  // per SM is what pays on these latency-bound kernels.
  bool fit = false;
  // Small n (the kept set capped, reading Q12c, so that every reduced system
  // has at most 64 rows) and a batch larger than the 4 CTAs/SM of path 1
  // hold: 64-thread CTAs (two warps per QP, one panel row per thread), up to
  // 8 per SM (128 registers per thread), so twice as many problems are in
  // flight.  Measured (one B200, 4096 problems): cbf7 620 K → 744 K QP/s,
  // cbf9 464 K → 571 K; one warp per QP (16 per SM) 726 K / 482 K.
  if (force_big) env_cap = -2;  // the fallback kernel of reading Q12c's guard: large-N layout
  if (formulation != QP_EXPLICIT && env_cap == -1 && !getenv("QPB200_FORCE_GLOBAL") && !getenv("QPB200_NO_SMALL") &&
      env_ctas == 0 && batch > 4 * sms) {
    const int need = std::min(L.Nmax, L.n4 + std::min(p, L.n4) + m);
    const int ncap = std::min(L.Nmax, 64);
    if (need <= ncap) {
      const size_t sm = path1_smem(L, m, p, ncap);
      const int ctas = std::min<int>(8, (int)(233472 / (sm + 1024)));
      if (ctas >= 6) {
        L.threads = 64; L.minb = 8; L.ncap = ncap; fit = true;
        L.pcap = std::min(p, ncap - L.n4 - m);
        if (const char* e = getenv("QPB200_PCAP")) L.pcap = std::max(0, std::min(L.pcap, atoi(e)));  // tests
        L.N4max = (ncap + 3) & ~3;
      }
    }
  }
  // Shapes whose worst case exceeds 256 rows also take path 1 when the
  // capped buffer (≤ 256 rows) still holds n4 + min(p, n4) + m (bezier4:
  // 110 K → 255 K QP/s at 4 CTAs/SM; bezier8: 25.6 K → 32.2 K at 1 CTA/SM of
  // 256 threads, against the large-N kernels); only larger systems need the
  // large-N kernels.
  if (!fit && env_cap == -1 && !getenv("QPB200_FORCE_GLOBAL")) {
    const int need = std::min(L.Nmax, L.n4 + std::min(p, L.n4) + m);
    const int want[4] = {4, 3, 2, 1};
    for (int w : want) {
      if (env_ctas && w != env_ctas) continue;
      int ncap = std::min(L.Nmax, 256);
      while (ncap >= need && path1_smem(L, m, p, ncap) > budget(w)) --ncap;
      if (ncap < need) continue;
      if (ncap < L.Nmax && getenv("QPB200_NO_PCAP")) continue;  // A/B: worst case only
      L.ncap = ncap; L.minb = w; fit = true;
      L.pcap = formulation == QP_EXPLICIT ? p : std::min(p, ncap - L.n4 - m);
      if (const char* e = getenv("QPB200_PCAP")) L.pcap = std::max(0, std::min(L.pcap, atoi(e)));  // tests
      L.N4max = (ncap + 3) & ~3;
      // at ≤ 2 CTAs/SM the registers allow 256 threads per QP (128 per thread
      // at 2 CTAs): config 3 73 K → 89 K QP/s
      if (w <= 2) L.threads = 256;
      break;
    }
  }
  if (!fit) {
    // large-N kernels: one CTA per SM (256 threads), tensor-core assembly,
    // the largest smem KKT buffer next to the vectors and the tc staging
    // area; iterations whose reduced system is larger use the CTA's global
    // workspace (hybrid)
    L.big = true;
    const size_t bud = budget(1);
    int lo = 0, hi = L.Nmax;
    if (smem_for(L, m, p, 0, true) > bud) {
      lo = 0;  // vectors alone do not fit: qp_create reports QP_ERR_SHAPE
    } else {
      while (lo < hi) {  // largest ncap that fits the budget
        const int mid = (lo + hi + 1) / 2;
        if (smem_for(L, m, p, mid, true) <= bud) lo = mid; else hi = mid - 1;
      }
    }
    L.ncap = lo;
    if (env_cap >= 0) L.ncap = std::min(env_cap, L.ncap);
    if (force_big) { L.threads = 256; L.minb = 1; L.batched = false; }
    if (getenv("QPB200_FORCE_GLOBAL")) L.ncap = 0;
    L.threads = 256; L.minb = 1;
    // the batched phase engine (path 4) unless the persistent large-N kernel
    // is asked for (A/B experiments, parity tests of that kernel)
    L.batched = formulation != QP_EXPLICIT && !getenv("QPB200_PERSISTENT_BIG") && !force_big;
  }
  if (L.batched) {
    // path 4: uniform packed layout (bnd_layout), the last 16-row block
    // allocated in full (the TMA boxes of bnd_tc_update read 16 rows)
    const qpb::KLayout K = qpb::KLayout::make(L.Nmax, L.n4, true);
    L.kglob = K.baseL + 16LL * K.Ll;
  }
  L.ksmem = L.ncap > 0 ? qpb::KLayout::make(L.ncap, L.n4).size() : 0;
  L.smem = qpb::ipm_smem_bytes(L.n4, m, p, L.N4max, L.ksmem, tc_floats(L.big), ro_ints(L, L.big));
  return L;
}

struct KernelSet {
  int threads;
  void (*solve)(const qpb::Args);
  void (*backward)(const qpb::Args);
};

KernelSet pick_kernels(const Layout& L, int formulation) {
  if (formulation == QP_EXPLICIT) {
    if (L.big) return {0, nullptr, nullptr};
    return {128, qpb::xpm_solve_kernel<128, 1>, qpb::xpm_backward_kernel<128, 1>};
  }
  if (L.big) return {256, qpb::ipm_kernel<256, 1, true>, qpb::ipm_kernel<256, 1, true>};
  if (L.threads == 64) return {64, qpb::ipm_kernel<64, 8, false, 64>, qpb::ipm_kernel<64, 8, false, 64>};
  if (L.threads == 256 && L.minb == 2) return {256, qpb::ipm_kernel<256, 2, false>, qpb::ipm_kernel<256, 2, false>};
  if (L.threads == 256) return {256, qpb::ipm_kernel<256, 1, false>, qpb::ipm_kernel<256, 1, false>};
  switch (L.minb) {
    case 4: return {128, qpb::ipm_kernel<128, 4, false>, qpb::ipm_kernel<128, 4, false>};
    case 3: return {128, qpb::ipm_kernel<128, 3, false>, qpb::ipm_kernel<128, 3, false>};
    default: return {128, qpb::ipm_kernel<128, 1, false>, qpb::ipm_kernel<128, 1, false>};
  }
}

bool aligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

}  // namespace

struct qp_ctx {
  qp_dims d;
  qp_config c;
  int device = 0;
  cudaStream_t stream = nullptr;
  Layout L{};
  KernelSet ks{};
  int ctas_per_sm = 0;
  bool solved = false;
  // pointers of the last solve (device memory)
  const float *Q = nullptr, *q = nullptr, *A = nullptr, *b = nullptr, *G = nullptr, *h = nullptr;
  float *x = nullptr, *s = nullptr, *z = nullptr, *y = nullptr;
  int32_t* status = nullptr;
  // owned device buffers
  int32_t* own_status = nullptr;  // forward status (kept for backward)
  float *wx = nullptr, *wy = nullptr, *wz = nullptr, *wdx = nullptr, *wdy = nullptr, *wdz = nullptr;
  // host-memory mode staging
  float *dQ_ = nullptr, *dq_ = nullptr, *dA_ = nullptr, *db_ = nullptr, *dG_ = nullptr, *dh_ = nullptr;
  float *dx_ = nullptr, *ds_ = nullptr, *dz_ = nullptr, *dy_ = nullptr, *ddl_ = nullptr;
  int32_t *dit_ = nullptr, *dst_ = nullptr;
  float *gQ_ = nullptr, *gq_ = nullptr, *gA_ = nullptr, *gb_ = nullptr, *gG_ = nullptr, *gh_ = nullptr;
  int64_t workspace = 0;
  int grid = 0;               // CTAs per launch (persistent over problems on path 2)
  float* kglob = nullptr;     // path 2 workspaces
  unsigned long long* prof = nullptr;  // QPB200_PHASE_PROFILE diagnostics
  // dynamic problem assignment and solve -> backward hand-off (path 1 and
  // large-N kernels): sched[0..15] solve launch counters, sched[16..31]
  // backward launch counters (one per pipeline chunk), zeroed by each solve;
  // done[b] = epoch of the last solve that finished problem b
  int* sched = nullptr;
  int* done = nullptr;
  unsigned long long* tl = nullptr;  // QPB200_TIMELINE diagnostics: [2][B][3]
  int epoch = 0;
  bool bwd_dirty = true;  // backward counters used since the last solve zeroed them
  // guarded chord relax (reading Q26): per problem the solve's cached factor,
  // its Jacobian block and a flag (allocated for the whole batch when enabled)
  float* kc = nullptr;
  long long kc_stride = 0;
  float* chd = nullptr;
  long long chd_stride = 0;
  int* chord_ok = nullptr;
  int chord_steps = 0;     // chord steps of the last backward (summed over the batch; path 4)
  int* chord_cnt = nullptr;  // device counter of the same (path 1)
  float* flops_solve = nullptr;        // per-problem algorithmic flops of the last calls
  float* flops_bwd = nullptr;
  // host-memory mode, path 1: the batch runs in kPipe chunks on their own
  // streams, so chunk i's kernel overlaps chunk i+1's H2D and chunk i−1's D2H
  // batched phase engine (path 4): per-problem state blocks and KKT
  // workspaces for `bchunk` problems at a time, the iteration counters
  float* bst = nullptr;
  long long bst_stride = 0;
  int bchunk = 0;
  int* bctl = nullptr;       // device: [0] problems factoring, [1] largest N4 among them, [2] chord steps, [3] caching
  int* hctl = nullptr;       // pinned host copy ([4 per lane])
  int nlanes = 1, lane_cap = 0;         // concurrent sub-batches of a chunk, problems per lane
  int sms = 148;                        // multiprocessors (persistent kr_gemm grid)
  int kr_div = 2;                       // kr_gemm grid = sms / kr_div (room for the other lane's kernels)
  cudaStream_t bstr[4] = {};            // lane streams (bstr[0] = the ctx stream at call time)
  cudaEvent_t bev[5] = {};              // ordering / read-back events
  int blaunch[2] = {0, 0};   // kernel launches of the last solve / backward
  // shared G: the assembly as one batched GEMM (kr_gemm.cuh)
  bool kr = false;
  float *whi = nullptr, *wlo = nullptr, *gghi = nullptr, *gglo = nullptr;
  int* slotmap = nullptr;
  float* dtg = nullptr;  // [bchunk][64·64] panel diagonal blocks (bnd_pdiag → bnd_prows)
  float* ug = nullptr;   // [bchunk][N4max·64] panel Schur updates (bnd_tc_update → bnd_pdiag / bnd_prows)
  char* tmaps = nullptr;  // device: one CUtensorMap per 16-row block of the KKT workspaces (bnd_tc_update_tma)
  // Q and G shared: residual GEMVs as batched GEMMs (bnd_sgemm), per problem [3][n4]
  float* pre = nullptr;
  long long off_x = 0, off_z = 0, off_t = 0, off_gx = 0, off_rhs = 0;  // state-block offsets (floats)
  int solve_nt = 128;    // threads of bnd_solve per problem
  int tma_stages = 0;     // 0: register-staged bnd_tc_update; else bnd_tc_update_tma<raw stages, operand buffers> as 10·S + NOB
  // reading Q12c guard (path 1 with a kept-set cap): problems whose capped
  // elimination would exceed fb_bound go to the uncapped large-N kernel,
  // launched (list-driven) right after each path-1 launch
  bool fb = false;
  float fb_bound = 0.f;
  Layout Lf{};
  int gridf = 0;
  float* kglobf = nullptr;
  int* fb_flag = nullptr;   // [B]
  int* fb_list = nullptr;   // [2B]: solve list, backward list (chunk segments at b0)
  int* fb_ctl = nullptr;    // [2][kPipe][2]: count, launch counter per call and chunk
  bool guard = false;                               // QPB200_GUARD: guard bands around workspaces
  std::vector<std::pair<char*, size_t>> guards;     // (allocation base, payload bytes)
  static constexpr int kPipe = 8;
  bool pipe = false;
  cudaStream_t pst[kPipe] = {};
  cudaEvent_t pev[kPipe + 1] = {};
};

namespace {

qp_err cuda_ok(cudaError_t e) { return e == cudaSuccess ? QP_OK : QP_ERR_CUDA; }

// Guard mode (QPB200_GUARD=1, tests: the memcheck substitute of
// tests/test_gpu_memcheck.py — compute-sanitizer is not available on the GPU
// pool): every workspace gets kGuard bytes of 0xFF before and after it;
// qp_debug_check_guards counts guard words a kernel overwrote.
constexpr size_t kGuard = 64 * 1024;

template <typename T>
qp_err dalloc(qp_ctx* c, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return QP_OK;
  if (c->guard) {
    char* base = nullptr;
    const size_t bytes = count * sizeof(T);
    if (cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuard) != cudaSuccess) return QP_ERR_OOM;
    if (cudaMemset(base, 0xFF, kGuard) != cudaSuccess || cudaMemset(base + kGuard + bytes, 0xFF, kGuard) != cudaSuccess)
      return QP_ERR_CUDA;
    c->guards.push_back({base, bytes});
    *p = reinterpret_cast<T*>(base + kGuard);
  } else if (cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)) != cudaSuccess) {
    return QP_ERR_OOM;
  }
  c->workspace += (int64_t)(count * sizeof(T));
  return QP_OK;
}

size_t field_elems(int64_t stride, int32_t B, size_t per) { return stride == 0 ? per : (size_t)B * per; }

void free_all(qp_ctx* c) {
  if (c->hctl) cudaFreeHost(c->hctl);
  void* ptrs[] = {c->pre, c->tmaps, c->kc, c->chd, c->chord_ok, c->chord_cnt, c->kglobf, c->fb_flag, c->fb_list, c->fb_ctl, c->ug, c->dtg, c->whi, c->wlo, c->gghi, c->gglo, c->slotmap, c->bst, c->bctl, c->tl, c->sched, c->done, c->kglob, c->flops_solve, c->flops_bwd, c->prof, c->own_status, c->wx, c->wy, c->wz, c->wdx, c->wdy, c->wdz, c->dQ_, c->dq_, c->dA_, c->db_,
                  c->dG_, c->dh_, c->dx_, c->ds_, c->dz_, c->dy_, c->ddl_, c->dit_, c->dst_, c->gQ_, c->gq_,
                  c->gA_, c->gb_, c->gG_, c->gh_};
  if (c->guard) {  // guard mode: the allocations start kGuard bytes before each pointer
    for (auto& g : c->guards) cudaFree(g.first);
    c->guards.clear();
    return;
  }
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

bool any_shared(const qp_dims& d) {
  return d.bstride_Q == 0 || d.bstride_q == 0 || d.bstride_A == 0 || d.bstride_b == 0 || d.bstride_G == 0 ||
         d.bstride_h == 0;
}

qpb::Args base_args(const qp_ctx* c) {
  qpb::Args a;
  std::memset(&a, 0, sizeof(a));
  a.B = c->d.batch; a.n = c->d.n; a.m = c->d.m_eq; a.p = c->d.p;
  a.n4 = c->L.n4; a.Nmax = c->L.Nmax; a.N4max = c->L.N4max;
  a.ksmem = c->L.ksmem; a.ncap = c->L.ncap; a.kglob_size = c->L.kglob;
  a.pcap = c->L.big ? c->d.p : c->L.pcap;
  a.tcf = tc_floats(c->L.big);
  a.rof = ro_ints(c->L, c->L.big);
  a.sQ = c->d.bstride_Q; a.sq = c->d.bstride_q; a.sA = c->d.bstride_A;
  a.sb = c->d.bstride_b; a.sG = c->d.bstride_G; a.sh = c->d.bstride_h;
  a.tol = c->c.tol; a.sigma = c->c.sigma; a.tau = c->c.tau; a.kappa_relax = c->c.kappa_relax;
  a.relax_ktol = c->c.relax_ktol; a.floor_rel = c->c.pivot_floor_rel; a.relax_tol = c->c.relax_tol;
  a.max_iter = c->c.max_iter; a.relax_max_iter = c->c.relax_max_iter;
  a.relax_mode = c->kc ? c->c.relax_mode : 0;
  a.chord_max = c->c.chord_max; a.chord_rho = c->c.chord_rho;
  a.kc = c->kc; a.kc_stride = c->kc_stride; a.chd = c->chd; a.chd_stride = c->chd_stride; a.chord_ok = c->chord_ok;
  a.chord_cnt = c->chord_cnt;
  return a;
}

// The arguments of problems [b0, b0 + nb) (shared fields have stride 0).
qpb::Args chunk_args(qpb::Args a, int b0, int nb) {
  const long long o = b0;
  const long long n = a.n, m = a.m, p = a.p;
  a.B = nb;
  a.Q += o * a.sQ; a.q += o * a.sq; a.A += o * a.sA; a.b += o * a.sb; a.G += o * a.sG; a.h += o * a.sh;
  a.x += o * n; a.y += o * m; a.z += o * p; a.s += o * p;
  if (a.iters) a.iters += o;
  if (a.status) a.status += o;
  if (a.status_out) a.status_out += o;
  if (a.done) a.done += o;
  if (a.dl) a.dl += o * n;
  if (a.gQ) a.gQ += o * n * n;
  if (a.gq) a.gq += o * n;
  if (a.gA) a.gA += o * m * n;
  if (a.gb) a.gb += o * m;
  if (a.gG) a.gG += o * p * n;
  if (a.gh) a.gh += o * p;
  if (a.wx) { a.wx += o * n; a.wdx += o * n; a.wy += o * m; a.wdy += o * m; a.wz += o * p; a.wdz += o * p; }
  if (a.riters) a.riters += o;
  if (a.rstatus) a.rstatus += o;
  if (a.flops) a.flops += o;
  if (a.fb_flag) a.fb_flag += o;
  if (a.fb_list) a.fb_list += o;
  if (a.prof) a.prof += 8 * o;
  if (a.kc) { a.kc += o * a.kc_stride; a.chd += o * a.chd_stride; a.chord_ok += o; }
  return a;
}

// m = 0 / p = 0 tensors may legitimately be NULL: point them at a dummy.
__device__ float g_dummy[4];

const float* nz(const float* p) {
  if (p) return p;
  void* d = nullptr;
  cudaGetSymbolAddress(&d, g_dummy);
  return static_cast<const float*>(d);
}

static qp_err h2d(qp_ctx* c, float* dst, const float* src, size_t count) {
  if (count == 0 || !src) return QP_OK;
  return cuda_ok(cudaMemcpyAsync(dst, src, count * sizeof(float), cudaMemcpyHostToDevice, c->stream));
}
template <typename T>
static qp_err d2h(qp_ctx* c, T* dst, const T* src, size_t count) {
  if (count == 0 || !dst) return QP_OK;
  return cuda_ok(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
}

// Reading Q12c guard: path-1 arguments of one launch (chunk ch; the list and
// its counters are per call and chunk).
void set_fb(const qp_ctx* c, qpb::Args& a, bool bwd, int ch) {
  if (!c->fb) return;
  a.fb_bound = c->fb_bound;
  a.fb_flag = c->fb_flag;
  a.fb_list = c->fb_list + (bwd ? c->d.batch : 0);
  a.fb_count = c->fb_ctl + 2 * (ch + (bwd ? qp_ctx::kPipe : 0));
}

// The fallback launch after a path-1 launch `ap` (chunk ch of nch, stream st):
// the uncapped large-N persistent kernel over the problems the path-1 launch
// handed over (list-driven; its CTAs exit at once when the list is empty).
qp_err launch_fallback(const qp_ctx* c, const qpb::Args& ap, bool bwd, int ch, int nch, cudaStream_t st) {
  if (!c->fb) return QP_OK;
  qpb::Args a = ap;
  const Layout& L = c->Lf;
  a.n4 = L.n4; a.Nmax = L.Nmax; a.N4max = L.N4max;
  a.ksmem = L.ksmem; a.ncap = L.ncap; a.kglob_size = L.kglob;
  a.pcap = c->d.p; a.tcf = qpb::tc::SMEM_BYTES / 4; a.rof = 0;
  a.fb_bound = 0.f; a.fb_flag = nullptr; a.fb_list = nullptr; a.fb_count = nullptr;
  a.plist = ap.fb_list;
  a.pcount = ap.fb_count;
  a.sched = ap.fb_count + 1;
  a.done = nullptr;  // stream-ordered after the path-1 launch: nothing to poll
  a.prof = nullptr; a.tl = nullptr;
  const int g = std::max(1, c->gridf / nch);
  a.kglob = c->kglobf + (size_t)ch * g * (size_t)L.kglob;  // this chunk's CTA workspaces
  qpb::ipm_kernel<256, 1, true><<<g, 256, L.smem, st>>>(a);
  return cuda_ok(cudaGetLastError());
}

constexpr int kBT = 128;  // threads of the batched-engine tensor-core / panel kernels
constexpr int kBS = 256;  // threads of the per-problem state kernels (resid, solve, update)
constexpr int kBW = 64;   // panel width of the batched factorisation

// smem attributes of the batched-engine kernels (once per process and shape)
qp_err bnd_setup(const qp_ctx* c) {
  const int sst = (int)(c->bst_stride * 4), ssv = (int)(c->L.N4max * 4);
  const int stc = qpb::tc::SMEM_BYTES;
  if (cudaFuncSetAttribute(qpb::bnd_begin<kBS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sst) ||
      cudaFuncSetAttribute(qpb::bnd_resid<kBS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sst) ||
      cudaFuncSetAttribute(qpb::bnd_resid<kBS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sst) ||
      cudaFuncSetAttribute(qpb::bnd_update<kBS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sst) ||
      cudaFuncSetAttribute(qpb::bnd_update<kBS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sst) ||
      cudaFuncSetAttribute(qpb::bnd_solve<kBT>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssv) ||
      cudaFuncSetAttribute(qpb::bnd_solve<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssv) ||
      cudaFuncSetAttribute(qpb::bnd_solve<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssv) ||
      cudaFuncSetAttribute(qpb::bnd_solve<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssv) ||
      cudaFuncSetAttribute(qpb::bnd_assemble<kBT>, cudaFuncAttributeMaxDynamicSharedMemorySize, stc) ||
      cudaFuncSetAttribute(qpb::bnd_tc_update<kBT>, cudaFuncAttributeMaxDynamicSharedMemorySize, stc) ||
      cudaFuncSetAttribute(qpb::bnd_tc_update_tma<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, qpb::tu::smem_bytes(2, 2)) ||
      cudaFuncSetAttribute(qpb::bnd_tc_update_tma<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, qpb::tu::smem_bytes(4, 2)) ||
      cudaFuncSetAttribute(qpb::kr::kr_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, qpb::kr::WS_SMEM_BYTES))
    return QP_ERR_CUDA;
  return QP_OK;
}

// TMA tensor maps of the batched engine's KKT workspaces (bnd_tc_update_tma):
// for every 16-row block b of the uniform packed layout (bnd_layout) a 3-D
// map {columns 16b + 20, rows 16, problems bchunk} with row stride (16b + 20)
// floats and problem stride kglob floats, 32 × 16 boxes, 128-byte swizzle.
qp_err make_tmaps(qp_ctx* c) {
  typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return QP_ERR_CUDA;
  const EncodeTiled encode = reinterpret_cast<EncodeTiled>(fn);
  const int NB = (c->L.N4max + 15) / 16;
  std::vector<CUtensorMap> maps(NB);
  for (int b = 0; b < NB; ++b) {
    const long long rl = 16LL * b + 20;
    void* gaddr = c->kglob + (128LL * b * (b + 1) + 64LL * b);
    const cuuint64_t dims[3] = {(cuuint64_t)rl, 16, (cuuint64_t)c->bchunk};
    const cuuint64_t strides[2] = {(cuuint64_t)(rl * 4), (cuuint64_t)(c->L.kglob * 4)};
    const cuuint32_t box[3] = {32, 16, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (encode(&maps[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, gaddr, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return QP_ERR_CUDA;
  }
  qp_err e;
  if ((e = dalloc(c, &c->tmaps, (size_t)NB * sizeof(CUtensorMap))) != QP_OK) return e;
  if (cudaMemcpy(c->tmaps, maps.data(), (size_t)NB * sizeof(CUtensorMap), cudaMemcpyHostToDevice) != cudaSuccess)
    return QP_ERR_CUDA;
  // opt-in (QPB200_TC_TMA = 42: four raw stages, two operand buffers; 22:
  // two and two): measured 2-3 % slower than the register-staged kernel on
  // config 4 and 8 % on config 5, so the default stays that
  c->tma_stages = 0;
  if (const char* e2 = getenv("QPB200_TC_TMA")) c->tma_stages = atoi(e2) == 22 ? 22 : 42;  // A/B
  return QP_OK;
}

// One call (solve: init + Alg. 1; backward: Alg. 2 + Alg. 3) on the batched
// phase engine: chunks of c->bchunk problems, per chunk the host loop over
// Newton iterations of bnd_kernels.cuh.  After bnd_resid the host reads back
// how many problems still iterate (and their largest padded system size,
// which bounds the panel loop), so the call returns once every problem has
// finished (the stream is synchronised at each iteration).
qp_err run_batched(qp_ctx* c, const qpb::Args& a0, bool bwd) {
  const int B = a0.B;
  const int n4 = c->L.n4, m = c->d.m_eq;
  const int T = (n4 + qpb::tc::TM - 1) / qpb::tc::TM;
  const int sst = (int)(c->bst_stride * 4), ssv = (int)(c->L.N4max * 4);
  const int stc = qpb::tc::SMEM_BYTES;
  const int krN = (qpb::kr::npairs(n4) + qpb::kr::BN - 1) / qpb::kr::BN;
  const size_t kpad = (size_t)qpb::kr::nkc(c->d.p) * qpb::kr::BK;
  int launches = 0;
  if (bwd) c->chord_steps = 0;
  // lanes: the chunk is split into c->nlanes sub-batches whose iteration
  // loops run interleaved on their own streams, so that one sub-batch's
  // phase kernels fill the tail waves of the other's
  c->bstr[0] = c->stream;
  cudaEvent_t ev0 = c->bev[0];
  if (cudaEventRecord(ev0, c->stream) != cudaSuccess) return QP_ERR_CUDA;
  for (int l = 1; l < c->nlanes; ++l)
    if (cudaStreamWaitEvent(c->bstr[l], ev0, 0) != cudaSuccess) return QP_ERR_CUDA;
  if (c->kr) {  // GG = the Khatri-Rao square of the shared G, once per call (lane 0; the others wait below)
    qpb::kr::kr_prep<<<4 * 148, 256, 0, c->stream>>>(a0.G, c->d.n, n4, c->d.p, c->gghi, c->gglo);
    ++launches;
    if (cudaEventRecord(ev0, c->stream) != cudaSuccess) return QP_ERR_CUDA;
    for (int l = 1; l < c->nlanes; ++l)
      if (cudaStreamWaitEvent(c->bstr[l], ev0, 0) != cudaSuccess) return QP_ERR_CUDA;
  }
  struct Lane {
    cudaStream_t st;
    qpb::BArgs ba;
    qpb::kr::GemmArgs ga;
    int nb, N4cur, k;
    bool live;
  };
  const int NL = c->nlanes, lcap = c->lane_cap;
  for (int b0 = 0; b0 < B; b0 += NL * lcap) {
    Lane ln[4];
    int nlive = 0;
    for (int l = 0; l < NL; ++l) {
      Lane& L = ln[l];
      const int lb0 = b0 + l * lcap;
      L.nb = std::max(0, std::min(lcap, B - lb0));
      L.live = L.nb > 0;
      if (!L.live) continue;
      ++nlive;
      L.st = c->bstr[l];
      qpb::BArgs& ba = L.ba;
      std::memset(&ba, 0, sizeof(ba));
      ba.a = chunk_args(a0, lb0, L.nb);
      ba.a.bwd = bwd ? 1 : 0;
      ba.st = c->bst + (size_t)l * lcap * c->bst_stride; ba.st_stride = c->bst_stride;
      ba.kw = c->kglob + (size_t)l * lcap * c->L.kglob; ba.kstride = c->L.kglob;
      ba.ctl = c->bctl + 4 * l;
      ba.ntiles = c->kr ? 0 : T * (T + 1) / 2;
      ba.w = kBW;
      ba.kr = c->kr ? 1 : 0;
      const size_t wrows = (size_t)((lcap + qpb::kr::BM - 1) / qpb::kr::BM) * qpb::kr::BM;
      ba.whi = c->whi ? c->whi + l * wrows * kpad : nullptr;
      ba.wlo = c->wlo ? c->wlo + l * wrows * kpad : nullptr;
      ba.slotmap = c->slotmap ? c->slotmap + (size_t)l * lcap : nullptr;
      ba.dtg = c->dtg + (size_t)l * lcap * 64 * 64;
      ba.ug = c->ug + (size_t)l * lcap * c->L.N4max * 64; ba.ustride = (long long)c->L.N4max * 64;
      ba.tmaps = c->tmaps; ba.lane_b0 = l * lcap;
      ba.pre = c->pre ? c->pre + (size_t)l * lcap * 3 * n4 : nullptr;
      ba.pre_stride = 3LL * n4;
      ba.fuse = getenv("QPB200_NO_FUSE") ? 0 : 1;
      qpb::kr::GemmArgs& ga = L.ga;
      if (c->kr) {
        ga.whi = ba.whi; ga.wlo = ba.wlo; ga.gghi = c->gghi; ga.gglo = c->gglo;
        ga.count = ba.ctl; ga.slotmap = ba.slotmap;
        ga.kw = ba.kw; ga.kstride = c->L.kglob; ga.st = ba.st; ga.st_stride = c->bst_stride;
        ga.Q = ba.a.Q; ga.sQ = ba.a.sQ;
        ga.n = c->d.n; ga.n4 = n4; ga.m = m; ga.p = c->d.p;
      }
      if (cudaMemsetAsync(ba.ctl, 0, 4 * sizeof(int), L.st) != cudaSuccess) return QP_ERR_CUDA;
      qpb::bnd_begin<kBS><<<L.nb, kBS, sst, L.st>>>(ba);
      ++launches;
      L.N4cur = bwd ? 0 : qpb::r4(n4 + m);  // the initial system (solve)
      L.k = bwd ? 0 : -1;
    }
    const int kmax = bwd ? c->c.relax_max_iter : c->c.max_iter;
    while (nlive > 0) {
      // residuals + stopping test of every live lane, then the read-backs
      for (int l = 0; l < NL; ++l) {
        Lane& L = ln[l];
        if (!L.live || L.k < 0) continue;
        if (cudaMemsetAsync(L.ba.ctl, 0, 4 * sizeof(int), L.st) != cudaSuccess) return QP_ERR_CUDA;
        L.ba.k = L.k;
        if (c->pre) {  // G x, Q x, Gᵀ z of every problem of the lane as three GEMMs
          const int n = c->d.n, p = c->d.p, mb = (L.nb + 63) / 64;
          const long long ss = c->bst_stride;
          float* st0 = L.ba.st;
          qpb::bnd_sgemm<true><<<dim3((p + 63) / 64, mb), 256, 0, L.st>>>(st0 + c->off_x, ss, a0.G, n,
                                                                            st0 + c->off_gx, ss, L.nb, p, n);
          qpb::bnd_sgemm<true><<<dim3((n + 63) / 64, mb), 256, 0, L.st>>>(st0 + c->off_x, ss, a0.Q, n, L.ba.pre,
                                                                            L.ba.pre_stride, L.nb, n, n);
          qpb::bnd_sgemm<false><<<dim3((n + 63) / 64, mb), 256, 0, L.st>>>(st0 + c->off_z, ss, a0.G, n,
                                                                             L.ba.pre + n4, L.ba.pre_stride, L.nb, n, p);
          launches += 3;
        }
        if (c->d.n >= 2 * kBS)  // column-quad GEMVs with 8 rows in flight (config 5)
          qpb::bnd_resid<kBS, true><<<L.nb, kBS, sst, L.st>>>(L.ba);
        else
          qpb::bnd_resid<kBS><<<L.nb, kBS, sst, L.st>>>(L.ba);
        ++launches;
        if (c->pre) {  // Gᵀ t (t: this iteration's right-hand-side vector of bnd_resid), added by bnd_solve
          const int n = c->d.n, p = c->d.p;
          qpb::bnd_sgemm<false><<<dim3((n + 63) / 64, (L.nb + 63) / 64), 256, 0, L.st>>>(
              L.ba.st + c->off_t, c->bst_stride, a0.G, n, L.ba.pre + 2 * n4, L.ba.pre_stride, L.nb, n, p);
          ++launches;
        }
        if (cudaMemcpyAsync(c->hctl + 4 * l, L.ba.ctl, 4 * sizeof(int), cudaMemcpyDeviceToHost, L.st) != cudaSuccess ||
            cudaEventRecord(c->bev[1 + l], L.st) != cudaSuccess)
          return QP_ERR_CUDA;
      }
      for (int l = 0; l < NL; ++l) {
        Lane& L = ln[l];
        if (!L.live) continue;
        // [0] problems that factor this iteration, [2] chord steps (reading
        // Q26: solve + update only), [3] problems caching their factor
        bool factor = true, cache = false;
        if (L.k >= 0) {
          if (cudaEventSynchronize(c->bev[1 + l]) != cudaSuccess) return QP_ERR_CUDA;
          if (c->hctl[4 * l] + c->hctl[4 * l + 2] == 0 || L.k > kmax + 1) { L.live = false; --nlive; continue; }
          L.N4cur = c->hctl[4 * l + 1];
          factor = c->hctl[4 * l] > 0;
          cache = c->hctl[4 * l + 3] > 0;
          if (bwd) c->chord_steps += c->hctl[4 * l + 2];
        }
        qpb::BArgs& ba = L.ba;
        cudaStream_t st = L.st;
        const int nb = L.nb;
        if (!factor) L.N4cur = 0;
        if (factor) {
        if (c->kr) qpb::bnd_scatter<kBS><<<nb, kBS, 0, st>>>(ba);
        else qpb::bnd_assemble<kBT><<<dim3(ba.ntiles + 1, nb), kBT, stc, st>>>(ba);
        ++launches;
        }
        if (factor && c->kr) {
          qpb::kr::kr_gemm<<<std::min(c->sms / c->kr_div, ((nb + qpb::kr::BM - 1) / qpb::kr::BM) * krN), qpb::kr::WS_THREADS,
                             qpb::kr::WS_SMEM_BYTES, st>>>(L.ga);
          ++launches;
        }
        for (int c0 = 0; c0 < L.N4cur; c0 += kBW) {
          ba.c0 = c0;
          if (c0 > 0) {
            const int tl = (L.N4cur - c0 + qpb::tc::TM - 1) / qpb::tc::TM;
            if (c->tma_stages) {
              // persistent, warp-specialised: one CTA per SM of this lane's share
              ba.ntiles_tu = tl;
              const long long items = (long long)tl * nb;
              const int grid = (int)std::min<long long>(items, std::max(1, c->sms / c->nlanes));
              const int v = c->tma_stages;  // raw stages × 10 + operand buffers
              const int S = v / 10, NOB = v % 10, sb = qpb::tu::smem_bytes(S, NOB);
              if (v == 22) qpb::bnd_tc_update_tma<2, 2><<<grid, qpb::TU_THREADS, sb, st>>>(ba);
              else qpb::bnd_tc_update_tma<4, 2><<<grid, qpb::TU_THREADS, sb, st>>>(ba);
            } else {
              qpb::bnd_tc_update<kBT><<<dim3(tl, nb), kBT, stc, st>>>(ba);
            }
            ++launches;
          }
          qpb::bnd_pdiag<32><<<nb, 32, 0, st>>>(ba);
          if (c0 + kBW < L.N4cur)
            qpb::bnd_prows<kBT><<<dim3((L.N4cur - c0 - kBW + kBT - 1) / kBT, nb), kBT, 0, st>>>(ba);
          launches += 2;
        }
        if (cache) {
          qpb::bnd_cache<kBT><<<dim3(8, nb), kBT, 0, st>>>(ba);
          ++launches;
        }
        if (c->solve_nt == 1024) qpb::bnd_solve<1024><<<nb, 1024, ssv, st>>>(ba);
        else if (c->solve_nt == 512) qpb::bnd_solve<512><<<nb, 512, ssv, st>>>(ba);
        else if (c->solve_nt == 256) qpb::bnd_solve<256><<<nb, 256, ssv, st>>>(ba);
        else qpb::bnd_solve<kBT><<<nb, kBT, ssv, st>>>(ba);
        if (c->pre) {  // G Δx (the solve's x part) of every problem: Δv recovery / the initial ẑ in bnd_update
          const int n = c->d.n, p = c->d.p;
          qpb::bnd_sgemm<true><<<dim3((p + 63) / 64, (nb + 63) / 64), 256, 0, st>>>(
              ba.st + c->off_rhs, c->bst_stride, a0.G, n, ba.st + c->off_gx, c->bst_stride, nb, p, n);
          ++launches;
        }
        if (c->d.n >= 2 * kBS)  // eight G rows in flight per warp (config 5)
          qpb::bnd_update<kBS, true><<<nb, kBS, sst, st>>>(ba);
        else
          qpb::bnd_update<kBS><<<nb, kBS, sst, st>>>(ba);
        launches += 2;
        ++L.k;
      }
    }
    if (cudaGetLastError() != cudaSuccess) return QP_ERR_CUDA;
  }
  // the ctx stream continues after every lane
  for (int l = 1; l < NL; ++l) {
    if (cudaEventRecord(c->bev[1 + l], c->bstr[l]) != cudaSuccess ||
        cudaStreamWaitEvent(c->stream, c->bev[1 + l], 0) != cudaSuccess)
      return QP_ERR_CUDA;
  }
  c->blaunch[bwd ? 1 : 0] = launches;
  return QP_OK;
}

}  // namespace

extern "C" {

qp_err qp_config_default(qp_config* cfg) {
  if (!cfg) return QP_ERR_INVALID_ARG;
  cfg->tol = 1e-5f;
  cfg->max_iter = 100;
  cfg->sigma = 0.1f;
  cfg->tau = 0.99f;
  cfg->kappa_relax = 1e-4f;
  cfg->relax_ktol = 1e-4f;
  cfg->relax_max_iter = 50;
  cfg->formulation = QP_IMPLICIT;
  cfg->pivot_floor_rel = 3.4526698e-4f;  // sqrt(FLT_EPSILON)
  cfg->mem_kind = QP_MEM_DEVICE;
  cfg->relax_tol = 1e-6f;
  cfg->relax_mode = QP_RELAX_CHORD;
  cfg->chord_max = 8;
  cfg->chord_rho = 0.5f;
  return QP_OK;
}

int32_t qp_max_kkt_dim(int32_t formulation) {
  (void)formulation;
  // path 1 (KKT in shared memory) up to ≈232; path 2 (KKT in a global
  // workspace) beyond, limited by the per-problem vectors in shared memory.
  return 4096;
}

const char* qp_error_string(qp_err e) {
  switch (e) {
    case QP_OK: return "ok";
    case QP_ERR_INVALID_ARG: return "invalid argument";
    case QP_ERR_SHAPE: return "unsupported shape";
    case QP_ERR_ALIGN: return "pointer not 4-byte aligned";
    case QP_ERR_CUDA: return "CUDA error";
    case QP_ERR_OOM: return "out of device memory";
    case QP_ERR_NOT_SOLVED: return "backward called before solve";
    case QP_ERR_UNSUPPORTED: return "unsupported option";
  }
  return "unknown error";
}

qp_err qp_create(qp_ctx** out, const qp_dims* d, const qp_config* cfg, int device, void* stream) {
  if (!out || !d) return QP_ERR_INVALID_ARG;
  *out = nullptr;
  if (d->batch < 1 || d->n < 1 || d->m_eq < 0 || d->p < 0) return QP_ERR_SHAPE;
  qp_config c;
  if (cfg) c = *cfg; else qp_config_default(&c);
  if (!(c.tol > 0.f) || c.max_iter < 0 || !(c.sigma > 0.f && c.sigma < 1.f) || !(c.tau > 0.f && c.tau <= 1.f) ||
      !(c.kappa_relax > 0.f) || !(c.relax_ktol > 0.f) || !(c.relax_tol > 0.f) || c.relax_max_iter < 0 || !(c.pivot_floor_rel >= 0.f) ||
      (c.formulation != QP_IMPLICIT && c.formulation != QP_EXPLICIT) ||
      (c.mem_kind != QP_MEM_DEVICE && c.mem_kind != QP_MEM_HOST && c.mem_kind != QP_MEM_HOST_ASYNC) ||
      (c.relax_mode != QP_RELAX_NEWTON && c.relax_mode != QP_RELAX_CHORD) || c.chord_max < 0 ||
      !(c.chord_rho > 0.f && c.chord_rho <= 1.f))
    return QP_ERR_INVALID_ARG;
  const int64_t strides[6] = {d->bstride_Q, d->bstride_q, d->bstride_A, d->bstride_b, d->bstride_G, d->bstride_h};
  const int64_t need[6] = {(int64_t)d->n * d->n, d->n, (int64_t)d->m_eq * d->n, d->m_eq, (int64_t)d->p * d->n,
                           d->p};
  for (int i = 0; i < 6; ++i) {
    if (strides[i] != 0 && strides[i] < need[i]) return QP_ERR_SHAPE;
    // host modes stage contiguous copies of the fields: padded batch strides
    // are a device-mode feature
    if (c.mem_kind != QP_MEM_DEVICE && strides[i] != 0 && strides[i] != need[i]) return QP_ERR_SHAPE;
  }
  Layout L = make_layout(d->n, d->m_eq, d->p, c.formulation);
  if (L.smem > kMaxSmem) return QP_ERR_SHAPE;  // vectors alone exceed the smem budget
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return QP_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return QP_ERR_CUDA;
  {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return QP_ERR_CUDA;
    L = make_layout(d->n, d->m_eq, d->p, c.formulation, d->batch, sms);
  }
  qp_ctx* ctx = new (std::nothrow) qp_ctx();
  if (!ctx) return QP_ERR_OOM;
  ctx->d = *d; ctx->c = c; ctx->device = device; ctx->stream = static_cast<cudaStream_t>(stream); ctx->L = L;
  ctx->guard = getenv("QPB200_GUARD") != nullptr;
  qp_err e = QP_OK;
  ctx->ks = pick_kernels(L, c.formulation);
  if (!ctx->ks.solve) { delete ctx; return QP_ERR_UNSUPPORTED; }  // standard arm: path 1 sizes only
  if (cudaFuncSetAttribute(ctx->ks.solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem) != cudaSuccess ||
      cudaFuncSetAttribute(ctx->ks.backward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem) !=
          cudaSuccess) {
    delete ctx;
    return QP_ERR_CUDA;
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->ctas_per_sm, ctx->ks.solve, ctx->ks.threads, L.smem);
  if (const char* e = getenv("QPB200_TC_W")) {  // experiments: tensor-core factorisation panel width
    const int w = atoi(e);
    cudaMemcpyToSymbol(qpb::g_tc_w, &w, sizeof(int));
  }
  // persistent CTAs (one KKT workspace each), looping over the batch
  {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    ctx->grid = std::min(d->batch, std::max(1, sms * std::max(1, ctx->ctas_per_sm)));
    const bool need_glob = L.big && L.ncap < L.Nmax && !L.batched;
    if (need_glob && (e = dalloc(ctx, &ctx->kglob, (size_t)ctx->grid * (size_t)L.kglob)) != QP_OK) {
      free_all(ctx); delete ctx; return e;
    }
  }
  if (!L.big && c.formulation == QP_IMPLICIT && L.pcap < d->p && !getenv("QPB200_NO_FALLBACK")) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    ctx->fb = true;
    ctx->fb_bound = 1e3f;
    if (const char* e2 = getenv("QPB200_FB_BOUND")) ctx->fb_bound = (float)atof(e2);  // tests
    ctx->Lf = make_layout(d->n, d->m_eq, d->p, c.formulation, d->batch, sms, true);
    ctx->gridf = sms;
    if (ctx->Lf.smem > kMaxSmem ||
        cudaFuncSetAttribute(qpb::ipm_kernel<256, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ctx->Lf.smem) != cudaSuccess) {
      free_all(ctx); delete ctx; return QP_ERR_CUDA;
    }
    if ((e = dalloc(ctx, &ctx->kglobf, (size_t)ctx->gridf * (size_t)ctx->Lf.kglob)) ||
        (e = dalloc(ctx, &ctx->fb_flag, (size_t)d->batch)) || (e = dalloc(ctx, &ctx->fb_list, 2 * (size_t)d->batch)) ||
        (e = dalloc(ctx, &ctx->fb_ctl, 4 * (size_t)qp_ctx::kPipe))) {
      free_all(ctx); delete ctx; return e;
    }
    if (cudaMemset(ctx->fb_flag, 0, sizeof(int) * d->batch) != cudaSuccess ||
        cudaMemset(ctx->fb_ctl, 0, sizeof(int) * 4 * qp_ctx::kPipe) != cudaSuccess) {
      free_all(ctx); delete ctx; return QP_ERR_CUDA;
    }
  }
  if (L.batched) {
    // per problem: a state block and a KKT workspace of capacity Nmax, for
    // up to half of the free device memory's worth of problems at a time
    ctx->bst_stride = qpb::bnd_state_floats(L.n4, d->m_eq, d->p, L.N4max);
    const size_t per = 4 * ((size_t)ctx->bst_stride + (size_t)L.kglob + 64 * 64 + (size_t)L.N4max * 64);
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    long long cap = (long long)(fr / 2 / per);
    if (const char* e2 = getenv("QPB200_BCHUNK")) cap = atoll(e2);  // tests: force several chunks
    ctx->bchunk = (int)std::max(1LL, std::min<long long>(d->batch, cap));
    // lanes: four for large systems (N ≥ 1024) in chunks of 256+ problems,
    // whose phase kernels alone fill few waves (config 5, 256 problems: 532 /
    // 564 / 577 / 583 QP/s with one / two / three / four); otherwise two for
    // chunks of 1184+ problems (config 4, 8192 problems: 42.4 K vs 41.8 K with
    // three, 40.9 K with four; 2048 problems: 39.1 K vs 37.9 K with one) and
    // one below (1024 problems: 30.9 K vs 30.7 K with two, 30.4 K with four)
    ctx->nlanes = (L.N4max >= 1024 && ctx->bchunk >= 256) ? 4 : ctx->bchunk >= 2 * 4 * 148 ? 2 : 1;
    if (const char* e2 = getenv("QPB200_BLANES")) ctx->nlanes = std::max(1, std::min(4, atoi(e2)));
    ctx->nlanes = std::min(ctx->nlanes, ctx->bchunk);
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
    ctx->kr_div = ctx->nlanes;
    if (const char* e2 = getenv("QPB200_KR_DIV")) ctx->kr_div = std::max(1, atoi(e2));  // A/B
    ctx->lane_cap = (ctx->bchunk + ctx->nlanes - 1) / ctx->nlanes;
    ctx->bchunk = ctx->lane_cap * ctx->nlanes;
    for (int l = 0; l < ctx->nlanes; ++l)
      if (l > 0 && cudaStreamCreateWithFlags(&ctx->bstr[l], cudaStreamNonBlocking) != cudaSuccess) {
        free_all(ctx); delete ctx; return QP_ERR_CUDA;
      }
    for (auto& ev : ctx->bev)
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) { free_all(ctx); delete ctx; return QP_ERR_CUDA; }
    if ((e = dalloc(ctx, &ctx->bst, (size_t)ctx->bchunk * ctx->bst_stride)) != QP_OK ||
        (e = dalloc(ctx, &ctx->kglob, (size_t)ctx->bchunk * (size_t)L.kglob)) != QP_OK ||
        (e = dalloc(ctx, &ctx->bctl, 16)) != QP_OK ||
        (e = dalloc(ctx, &ctx->dtg, (size_t)ctx->bchunk * 64 * 64)) != QP_OK ||
        (e = dalloc(ctx, &ctx->ug, (size_t)ctx->bchunk * L.N4max * 64)) != QP_OK) {
      free_all(ctx); delete ctx; return e;
    }
    if (cudaMallocHost(&ctx->hctl, 16 * sizeof(int)) != cudaSuccess || bnd_setup(ctx) != QP_OK) {
      free_all(ctx); delete ctx; return QP_ERR_CUDA;
    }
    if (getenv("QPB200_TC_TMA") && (e = make_tmaps(ctx)) != QP_OK) { free_all(ctx); delete ctx; return e; }
    // triangular solves of large systems: more threads per problem keep more
    // factor rows in flight (config 5, N ≈ 1.7-3 K: 560 → 609 QP/s at 512;
    // config 4, N ≈ 340: 128 stays, 256 is 5 % slower)
    ctx->solve_nt = L.N4max >= 1024 ? 512 : 128;
    if (const char* e2 = getenv("QPB200_SOLVE_NT")) ctx->solve_nt = atoi(e2);
    // shared G: the assembly runs as one GEMM over the batch (kr_gemm.cuh)
    ctx->kr = d->bstride_G == 0 && d->p > 0 && !getenv("QPB200_NO_KR");
    // shared Q and G: the residual GEMVs as batched GEMMs too (bnd_sgemm)
    if (ctx->kr && d->bstride_Q == 0 && !getenv("QPB200_NO_PRE")) {
      if ((e = dalloc(ctx, &ctx->pre, (size_t)ctx->bchunk * 3 * L.n4)) != QP_OK) { free_all(ctx); delete ctx; return e; }
      const qpb::Smem S0 = qpb::layout(nullptr, L.n4, d->m_eq, d->p, L.N4max, 0, 0, 0);
      ctx->off_x = 16 + (S0.x - (float*)nullptr); ctx->off_z = 16 + (S0.z - (float*)nullptr);
      ctx->off_t = 16 + (S0.t - (float*)nullptr); ctx->off_gx = 16 + (S0.gx - (float*)nullptr);
      ctx->off_rhs = 16 + (S0.rhs - (float*)nullptr);
    }
    if (ctx->kr) {
      const size_t kpad = (size_t)qpb::kr::nkc(d->p) * qpb::kr::BK;
      const size_t mrows = (size_t)ctx->nlanes * ((ctx->lane_cap + qpb::kr::BM - 1) / qpb::kr::BM) * qpb::kr::BM;
      const size_t nrows = (size_t)((qpb::kr::npairs(L.n4) + qpb::kr::BN - 1) / qpb::kr::BN) * qpb::kr::BN;
      if ((e = dalloc(ctx, &ctx->whi, mrows * kpad)) || (e = dalloc(ctx, &ctx->wlo, mrows * kpad)) ||
          (e = dalloc(ctx, &ctx->gghi, nrows * kpad)) || (e = dalloc(ctx, &ctx->gglo, nrows * kpad)) ||
          (e = dalloc(ctx, &ctx->slotmap, ctx->bchunk))) {
        free_all(ctx); delete ctx; return e;
      }
    }
  }
  // guarded chord relax (reading Q26): a cached factor per problem of the
  // whole batch (path 4: the packed workspace; path 1: the shared-memory KKT
  // buffer's contents), when it fits in a quarter of the free device memory
  // (otherwise the relax stays exact Newton: qp_info.relax_mode says which)
  if (c.relax_mode == QP_RELAX_CHORD && c.formulation == QP_IMPLICIT && d->p > 0 && (L.batched || !L.big)) {
    size_t fr2 = 0, tot2 = 0;
    cudaMemGetInfo(&fr2, &tot2);
    const long long ks = L.batched ? (long long)L.kglob : (long long)((L.ksmem + 3) & ~3);
    const long long cs = qpb::chd_floats(d->p, L.N4max);
    const size_t need = (size_t)d->batch * 4 * ((size_t)ks + (size_t)cs + 1);
    if (need <= fr2 / 4) {
      ctx->kc_stride = ks; ctx->chd_stride = cs;
      if ((e = dalloc(ctx, &ctx->kc, (size_t)d->batch * (size_t)ks)) ||
          (e = dalloc(ctx, &ctx->chd, (size_t)d->batch * (size_t)cs)) || (e = dalloc(ctx, &ctx->chord_ok, (size_t)d->batch)) ||
          (e = dalloc(ctx, &ctx->chord_cnt, 1))) {
        free_all(ctx); delete ctx; return e;
      }
      if (cudaMemset(ctx->chord_ok, 0, sizeof(int) * d->batch) != cudaSuccess) { free_all(ctx); delete ctx; return QP_ERR_CUDA; }
    }
  }
  const int B = d->batch, n = d->n, m = d->m_eq, p = d->p;
  if ((e = dalloc(ctx, &ctx->own_status, B)) || (e = dalloc(ctx, &ctx->flops_solve, B)) ||
      (e = dalloc(ctx, &ctx->flops_bwd, B)) || (e = dalloc(ctx, &ctx->sched, 32)) ||
      (e = dalloc(ctx, &ctx->done, std::max(B, 1)))) {
    free_all(ctx); delete ctx; return e;
  }
  if (cudaMemset(ctx->done, 0, sizeof(int) * std::max(B, 1)) != cudaSuccess) {  // epochs start at 1
    free_all(ctx); delete ctx; return QP_ERR_CUDA;
  }
  if (any_shared(*d)) {
    if ((e = dalloc(ctx, &ctx->wx, (size_t)B * n)) || (e = dalloc(ctx, &ctx->wdx, (size_t)B * n)) ||
        (e = dalloc(ctx, &ctx->wy, (size_t)B * m)) || (e = dalloc(ctx, &ctx->wdy, (size_t)B * m)) ||
        (e = dalloc(ctx, &ctx->wz, (size_t)B * p)) || (e = dalloc(ctx, &ctx->wdz, (size_t)B * p))) {
      free_all(ctx); delete ctx; return e;
    }
  }
  if (c.mem_kind != QP_MEM_DEVICE) {
    if ((e = dalloc(ctx, &ctx->dQ_, field_elems(d->bstride_Q, B, (size_t)n * n))) ||
        (e = dalloc(ctx, &ctx->dq_, field_elems(d->bstride_q, B, n))) ||
        (e = dalloc(ctx, &ctx->dA_, field_elems(d->bstride_A, B, (size_t)m * n))) ||
        (e = dalloc(ctx, &ctx->db_, field_elems(d->bstride_b, B, m))) ||
        (e = dalloc(ctx, &ctx->dG_, field_elems(d->bstride_G, B, (size_t)p * n))) ||
        (e = dalloc(ctx, &ctx->dh_, field_elems(d->bstride_h, B, p))) ||
        (e = dalloc(ctx, &ctx->dx_, (size_t)B * n)) || (e = dalloc(ctx, &ctx->ds_, (size_t)B * p)) ||
        (e = dalloc(ctx, &ctx->dz_, (size_t)B * p)) || (e = dalloc(ctx, &ctx->dy_, (size_t)B * m)) ||
        (e = dalloc(ctx, &ctx->ddl_, (size_t)B * n)) || (e = dalloc(ctx, &ctx->dit_, B)) ||
        (e = dalloc(ctx, &ctx->dst_, B)) ||
        (e = dalloc(ctx, &ctx->gQ_, field_elems(d->bstride_Q, B, (size_t)n * n))) ||
        (e = dalloc(ctx, &ctx->gq_, field_elems(d->bstride_q, B, n))) ||
        (e = dalloc(ctx, &ctx->gA_, field_elems(d->bstride_A, B, (size_t)m * n))) ||
        (e = dalloc(ctx, &ctx->gb_, field_elems(d->bstride_b, B, m))) ||
        (e = dalloc(ctx, &ctx->gG_, field_elems(d->bstride_G, B, (size_t)p * n))) ||
        (e = dalloc(ctx, &ctx->gh_, field_elems(d->bstride_h, B, p)))) {
      free_all(ctx); delete ctx; return e;
    }
    // chunked copy/compute overlap: path 1 only (the chunk kernels run
    // concurrently; the global KKT workspaces of paths 2/3 are per CTA slot)
    if (!ctx->kglob && B >= 2 * 64 && !getenv("QPB200_NO_PIPE")) {
      bool ok = true;
      for (auto& st : ctx->pst) ok = ok && cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess;
      for (auto& ev : ctx->pev) ok = ok && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
      ctx->pipe = ok;
    }
  }
  *out = ctx;
  return QP_OK;
}

qp_err qp_set_stream(qp_ctx* c, void* stream) {
  if (!c) return QP_ERR_INVALID_ARG;
  c->stream = static_cast<cudaStream_t>(stream);
  return QP_OK;
}

qp_err qp_get_info(const qp_ctx* c, qp_info* info) {
  if (!c || !info) return QP_ERR_INVALID_ARG;
  info->path = !c->L.big ? 1 : c->L.batched ? 4 : (c->L.ncap > 0 ? 3 : 2);  // 1 smem, 2 global, 3 hybrid, 4 batched
  info->partition_cap = c->L.big ? c->d.p : c->L.pcap;
  info->threads = c->ks.threads;
  info->smem_bytes = (int32_t)c->L.smem;
  info->ctas_per_sm = c->ctas_per_sm;
  info->kkt_dim = c->L.Nmax;
  info->launches_solve = 1;
  const qp_dims& d = c->d;
  int extra = 0;
  if (d.bstride_Q == 0) ++extra;
  if (d.bstride_q == 0) ++extra;
  if (d.bstride_A == 0 && d.m_eq > 0) ++extra;
  if (d.bstride_b == 0 && d.m_eq > 0) ++extra;
  if (d.bstride_G == 0 && d.p > 0) ++extra;
  if (d.bstride_h == 0 && d.p > 0) ++extra;
  info->launches_backward = 1 + extra;
  if (c->L.batched) {  // phase kernels: counted by the last calls
    info->launches_solve = c->blaunch[0];
    info->launches_backward = c->blaunch[1] + extra;
    info->threads = kBS;
    info->smem_bytes = (int32_t)(c->bst_stride * 4);  // state block of the per-problem phases
    info->ctas_per_sm = 0;                            // varies by phase kernel
  }
  info->workspace_bytes = c->workspace;
  info->relax_mode = c->kc ? c->c.relax_mode : QP_RELAX_NEWTON;
  info->chord_steps = c->chord_steps;
  if (c->chord_cnt && !c->L.batched) {  // path 1: the device counter of the last backward
    if (cudaStreamSynchronize(c->stream) != cudaSuccess ||
        cudaMemcpy(&info->chord_steps, c->chord_cnt, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
      return QP_ERR_CUDA;
  }
  info->handed_solve = info->handed_backward = 0;
  if (c->fb) {  // reading Q12c guard: hand-over counts of the last calls (all chunks)
    int h[4 * qp_ctx::kPipe];
    if (cudaStreamSynchronize(c->stream) != cudaSuccess ||
        cudaMemcpy(h, c->fb_ctl, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess)
      return QP_ERR_CUDA;
    for (int ch = 0; ch < qp_ctx::kPipe; ++ch) {
      info->handed_solve += h[2 * ch];
      info->handed_backward += h[2 * (ch + qp_ctx::kPipe)];
    }
  }
  return QP_OK;
}

qp_err qp_solve_batched(qp_ctx* c, const float* Q, const float* q, const float* A, const float* b, const float* G,
                        const float* h, float* x, float* s, float* z, float* y, int32_t* iters, int32_t* status) {
  if (!c) return QP_ERR_INVALID_ARG;
  const qp_dims& d = c->d;
  const int B = d.batch, n = d.n, m = d.m_eq, p = d.p;
  if (!Q || !q || !x || !iters || !status || (m > 0 && (!A || !b || !y)) || (p > 0 && (!G || !h || !s || !z)))
    return QP_ERR_INVALID_ARG;
  const void* ptrs[] = {Q, q, A, b, G, h, x, s, z, y, iters, status};
  for (const void* pp : ptrs)
    if (pp && !aligned4(pp)) return QP_ERR_ALIGN;
  if (cudaSetDevice(c->device) != cudaSuccess) return QP_ERR_CUDA;
  qp_err e;
  const bool host = c->c.mem_kind != QP_MEM_DEVICE;
  const bool hsync = c->c.mem_kind == QP_MEM_HOST;  // QP_MEM_HOST_ASYNC: the caller synchronises
  // host mode: device copies of the six fields (stride 0 = shared, one copy)
  float* const stage[6] = {c->dQ_, c->dq_, c->dA_, c->db_, c->dG_, c->dh_};
  const float* const src[6] = {Q, q, A, b, G, h};
  const int64_t bstr[6] = {d.bstride_Q, d.bstride_q, d.bstride_A, d.bstride_b, d.bstride_G, d.bstride_h};
  const size_t per[6] = {(size_t)n * n, (size_t)n, (size_t)m * n, (size_t)m, (size_t)p * n, (size_t)p};
  const bool pipe = host && c->pipe;
  if (host) {
    for (int f = 0; f < 6; ++f)
      if (!pipe || bstr[f] == 0)  // pipelined: per-problem fields go chunk by chunk below
        if ((e = h2d(c, stage[f], src[f], field_elems(bstr[f], B, per[f]))) != QP_OK) return e;
    c->Q = c->dQ_; c->q = c->dq_; c->A = c->dA_; c->b = c->db_; c->G = c->dG_; c->h = c->dh_;
    c->x = c->dx_; c->s = c->ds_; c->z = c->dz_; c->y = c->dy_;
  } else {
    c->Q = Q; c->q = q; c->A = A; c->b = b; c->G = G; c->h = h;
    c->x = x; c->s = s; c->z = z; c->y = y;
  }
  qpb::Args a = base_args(c);
  a.Q = nz(c->Q); a.q = nz(c->q); a.A = nz(c->A); a.b = nz(c->b); a.G = nz(c->G); a.h = nz(c->h);
  float* dummy = const_cast<float*>(nz(nullptr));
  a.x = c->x; a.y = c->y ? c->y : dummy; a.z = c->z ? c->z : dummy; a.s = c->s ? c->s : dummy;
  a.iters = host ? c->dit_ : iters;
  a.status = c->own_status;
  a.status_out = host ? nullptr : status;
  const bool implicit = c->c.formulation != QP_EXPLICIT;
  if (implicit) {
    // zero every launch counter of this solve and of the backward that follows
    c->solved = false;  // a backward must not wait on an epoch whose solve was never launched
    if ((e = cuda_ok(cudaMemsetAsync(c->sched, 0, sizeof(int) * 32, c->stream))) != QP_OK) return e;
    c->bwd_dirty = false;
    a.sched = c->sched;
    a.done = c->done;
    a.epoch = ++c->epoch;
    if (getenv("QPB200_TIMELINE") && !c->tl) cudaMalloc(&c->tl, sizeof(unsigned long long) * 6 * (size_t)B);
    a.tl = c->tl;
  }
  if (getenv("QPB200_PHASE_PROFILE") && !c->prof) {
    cudaMalloc(&c->prof, sizeof(unsigned long long) * 8 * B);
    int on = 1;
    cudaMemcpyToSymbol(qpb::g_fac_on, &on, sizeof(int));
  }
  if (c->prof) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbolAsync(qpb::g_fac_cycles, z, sizeof(z), 0, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyToSymbolAsync(qpb::g_tcf_cycles, z, sizeof(z), 0, cudaMemcpyHostToDevice, c->stream);
  }
  a.prof = c->prof;
  a.flops = c->flops_solve;
  a.kglob = c->kglob;
  if (implicit) set_fb(c, a, false, 0);
  if (pipe) {
    // chunk ch on stream pst[ch]: H2D of its problems, its kernel, D2H of its outputs
    constexpr int KP = qp_ctx::kPipe;
    const int cs = (B + KP - 1) / KP;
    if ((e = cuda_ok(cudaEventRecord(c->pev[KP], c->stream))) != QP_OK) return e;
    for (int ch = 0; ch < KP; ++ch) {
      const int b0 = ch * cs, nb = std::min(cs, B - b0);
      if (nb <= 0) break;
      cudaStream_t st = c->pst[ch];
      if ((e = cuda_ok(cudaStreamWaitEvent(st, c->pev[KP], 0))) != QP_OK) return e;
      for (int f = 0; f < 6; ++f)
        if (bstr[f] != 0 && per[f] > 0 &&
            (e = cuda_ok(cudaMemcpyAsync(stage[f] + (size_t)b0 * bstr[f], src[f] + (size_t)b0 * bstr[f],
                                         sizeof(float) * (size_t)nb * bstr[f], cudaMemcpyHostToDevice, st))) !=
                QP_OK)
          return e;
      qpb::Args ac = chunk_args(a, b0, nb);
      if (implicit) ac.sched = c->sched + ch;
      if (c->fb) {
        ac.fb_count = c->fb_ctl + 2 * ch;
        if ((e = cuda_ok(cudaMemsetAsync(ac.fb_count, 0, 2 * sizeof(int), st))) != QP_OK) return e;
      }
      c->ks.solve<<<std::min(c->grid, nb), c->ks.threads, c->L.smem, st>>>(ac);
      if ((e = cuda_ok(cudaGetLastError())) != QP_OK) return e;
      if ((e = launch_fallback(c, ac, false, ch, KP, st)) != QP_OK) return e;
      auto o2h = [&](auto* dst, const auto* dsrc, size_t per_prob) -> qp_err {
        if (!dst || per_prob == 0) return QP_OK;
        return cuda_ok(cudaMemcpyAsync(dst + (size_t)b0 * per_prob, dsrc + (size_t)b0 * per_prob,
                                       sizeof(*dst) * (size_t)nb * per_prob, cudaMemcpyDeviceToHost, st));
      };
      if ((e = o2h(x, c->dx_, n)) || (e = o2h(s, c->ds_, p)) || (e = o2h(z, c->dz_, p)) ||
          (e = o2h(y, c->dy_, m)) || (e = o2h(iters, c->dit_, 1)) || (e = o2h(status, c->own_status, 1)))
        return e;
      if ((e = cuda_ok(cudaEventRecord(c->pev[ch], st))) != QP_OK) return e;
      if ((e = cuda_ok(cudaStreamWaitEvent(c->stream, c->pev[ch], 0))) != QP_OK) return e;
    }
    if (hsync && (e = cuda_ok(cudaStreamSynchronize(c->stream))) != QP_OK) return e;
  } else if (c->L.batched) {
    if ((e = run_batched(c, a, false)) != QP_OK) return e;
  } else {
    if (c->fb && (e = cuda_ok(cudaMemsetAsync(a.fb_count, 0, 2 * sizeof(int), c->stream))) != QP_OK) return e;
    c->ks.solve<<<c->grid, c->ks.threads, c->L.smem, c->stream>>>(a);
    if ((e = cuda_ok(cudaGetLastError())) != QP_OK) return e;
    if ((e = launch_fallback(c, a, false, 0, 1, c->stream)) != QP_OK) return e;
  }
  if (pipe) {
    // outputs already copied chunk by chunk
  } else if (host) {
    if ((e = d2h(c, x, c->dx_, (size_t)B * n)) || (e = d2h(c, s, c->ds_, (size_t)B * p)) ||
        (e = d2h(c, z, c->dz_, (size_t)B * p)) || (e = d2h(c, y, c->dy_, (size_t)B * m)) ||
        (e = d2h(c, iters, c->dit_, (size_t)B)) || (e = d2h(c, status, c->own_status, (size_t)B)))
      return e;
    if (hsync && (e = cuda_ok(cudaStreamSynchronize(c->stream))) != QP_OK) return e;
  } else if (!implicit) {
    if ((e = cuda_ok(cudaMemcpyAsync(status, c->own_status, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice,
                                     c->stream))) != QP_OK)
      return e;
  }  // (implicit kernels write the caller's status array themselves)
  c->solved = true;
  if (c->prof) {
    cudaStreamSynchronize(c->stream);
    unsigned long long* hp = new unsigned long long[8 * (size_t)B];
    cudaMemcpy(hp, c->prof, sizeof(unsigned long long) * 8 * B, cudaMemcpyDeviceToHost);
    double tot[8] = {0};
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < 8; ++j) tot[j] += (double)hp[i * 8 + j];
    fprintf(stderr, "[qpb200 phase cycles per CTA] resid %.0f assemble %.0f factor %.0f solve %.0f update %.0f"
                    " | sum pa %.1f sum N %.1f\n",
            tot[0] / B, tot[1] / B, tot[2] / B, tot[3] / B, tot[4] / B, tot[5] / B, tot[6] / B);
    {
      std::vector<unsigned long long> mx(B);
      for (int i = 0; i < B; ++i) mx[i] = hp[i * 8 + 7];
      std::sort(mx.begin(), mx.end());
      fprintf(stderr, "[qpb200 largest reduced system per problem] median %llu p90 %llu p99 %llu max %llu (Nmax %d)\n",
              mx[B / 2], mx[(size_t)(0.9 * (B - 1))], mx[(size_t)(0.99 * (B - 1))], mx[B - 1], c->L.Nmax);
    }
    delete[] hp;
    unsigned long long fc[4];
    cudaMemcpyFromSymbol(fc, qpb::g_fac_cycles, sizeof(fc));
    if (fc[3]) fprintf(stderr, "[qpb200 factor sub-phases per factorisation] panel %.0f syrk %.0f inverses %.0f\n",
                       (double)fc[0] / fc[3], (double)fc[1] / fc[3], (double)fc[2] / fc[3]);
    cudaMemcpyFromSymbol(fc, qpb::g_tcf_cycles, sizeof(fc));
    if (fc[3])
      fprintf(stderr, "[qpb200 tensor-core factorisations: %llu] tc updates %.0f panels %.0f inverses %.0f cycles each\n",
              fc[3], (double)fc[0] / fc[3], (double)fc[1] / fc[3], (double)fc[2] / fc[3]);
  }
  return QP_OK;
}

qp_err qp_backward_batched(qp_ctx* c, const float* dl_dx, float* dQ, float* dq, float* dA, float* db, float* dG,
                           float* dh, int32_t* relax_iters, int32_t* status) {
  if (!c || !dl_dx) return QP_ERR_INVALID_ARG;
  if (!c->solved) return QP_ERR_NOT_SOLVED;
  const void* ptrs[] = {dl_dx, dQ, dq, dA, db, dG, dh, relax_iters, status};
  for (const void* pp : ptrs)
    if (pp && !aligned4(pp)) return QP_ERR_ALIGN;
  if (cudaSetDevice(c->device) != cudaSuccess) return QP_ERR_CUDA;
  const qp_dims& d = c->d;
  const int B = d.batch, n = d.n, m = d.m_eq, p = d.p;
  const bool host = c->c.mem_kind != QP_MEM_DEVICE;
  const bool hsync = c->c.mem_kind == QP_MEM_HOST;  // QP_MEM_HOST_ASYNC: the caller synchronises
  qp_err e;
  const float* dl = dl_dx;
  float *oQ = dQ, *oq = dq, *oA = dA, *ob = db, *oG = dG, *oh = dh;
  int32_t *oit = relax_iters, *ost = status;
  const bool pipe = host && c->pipe;
  if (host) {
    if (!pipe && (e = h2d(c, c->ddl_, dl_dx, (size_t)B * n)) != QP_OK) return e;
    dl = c->ddl_;
    oQ = dQ ? c->gQ_ : nullptr; oq = dq ? c->gq_ : nullptr; oA = dA ? c->gA_ : nullptr;
    ob = db ? c->gb_ : nullptr; oG = dG ? c->gG_ : nullptr; oh = dh ? c->gh_ : nullptr;
    oit = c->dit_; ost = c->dst_;
  }
  qpb::Args a = base_args(c);
  a.Q = nz(c->Q); a.q = nz(c->q); a.A = nz(c->A); a.b = nz(c->b); a.G = nz(c->G); a.h = nz(c->h);
  float* dummy = const_cast<float*>(nz(nullptr));
  a.x = c->x; a.y = c->y ? c->y : dummy; a.z = c->z ? c->z : dummy; a.s = c->s ? c->s : dummy;
  a.status = c->own_status;
  a.dl = dl;
  a.bwd = 1;
  // per-problem gradients for non-shared fields; shared fields via batch sums
  a.gQ = d.bstride_Q ? oQ : nullptr;
  a.gq = d.bstride_q ? oq : nullptr;
  a.gA = (d.bstride_A && m > 0) ? oA : nullptr;
  a.gb = (d.bstride_b && m > 0) ? ob : nullptr;
  a.gG = (d.bstride_G && p > 0) ? oG : nullptr;
  a.gh = (d.bstride_h && p > 0) ? oh : nullptr;
  const bool shared = any_shared(d);
  if (shared) {
    a.wx = c->wx; a.wdx = c->wdx;
    a.wy = m ? c->wy : dummy; a.wdy = m ? c->wdy : dummy;
    a.wz = p ? c->wz : dummy; a.wdz = p ? c->wdz : dummy;
  }
  a.riters = oit;
  a.rstatus = ost;
  a.flops = c->flops_bwd;
  a.kglob = c->kglob;
  const bool implicit = c->c.formulation != QP_EXPLICIT;
  if (implicit) set_fb(c, a, true, 0);
  if (implicit) {
    if (c->bwd_dirty &&
        (e = cuda_ok(cudaMemsetAsync(c->sched + 16, 0, sizeof(int) * 16, c->stream))) != QP_OK)
      return e;
    c->bwd_dirty = true;
    a.sched = c->sched + 16;
    a.done = c->done;
    a.epoch = c->epoch;
    a.tl = c->tl ? c->tl + 3 * (size_t)B : nullptr;
  }
  // chord-step counter (diagnostic; with QP_MEM_HOST_ASYNC the chunks are not
  // ordered after this reset, so the count is approximate there)
  if (c->chord_cnt && (e = cuda_ok(cudaMemsetAsync(c->chord_cnt, 0, sizeof(int), c->stream))) != QP_OK) return e;
  if (pipe) {
    // chunk ch on stream pst[ch]: H2D of its cotangents, its kernel, D2H of its
    // per-problem gradients; shared-field sums follow on c->stream
    constexpr int KP = qp_ctx::kPipe;
    const int cs = (B + KP - 1) / KP;
    if ((e = cuda_ok(cudaEventRecord(c->pev[KP], c->stream))) != QP_OK) return e;
    float* const gdev[6] = {a.gQ, a.gq, a.gA, a.gb, a.gG, a.gh};
    float* const ghost[6] = {dQ, dq, dA, db, dG, dh};
    const size_t gper[6] = {(size_t)n * n, (size_t)n, (size_t)m * n, (size_t)m, (size_t)p * n, (size_t)p};
    for (int ch = 0; ch < KP; ++ch) {
      const int b0 = ch * cs, nb = std::min(cs, B - b0);
      if (nb <= 0) break;
      cudaStream_t st = c->pst[ch];
      // QP_MEM_HOST: after all earlier work on the ctx stream.  QP_MEM_HOST_ASYNC:
      // chunk ch follows the solve's chunk ch on its own stream only, so the
      // first backward chunks overlap the last solve chunks
      if (hsync && (e = cuda_ok(cudaStreamWaitEvent(st, c->pev[KP], 0))) != QP_OK) return e;
      if ((e = cuda_ok(cudaMemcpyAsync(c->ddl_ + (size_t)b0 * n, dl_dx + (size_t)b0 * n, sizeof(float) * (size_t)nb * n,
                                       cudaMemcpyHostToDevice, st))) != QP_OK)
        return e;
      qpb::Args ac = chunk_args(a, b0, nb);
      if (implicit) {
        // this chunk's problem counter, zeroed on the chunk's own stream: with
        // QP_MEM_HOST_ASYNC the chunk is ordered only after the work on pst[ch]
        // (the solve chunk, an earlier backward chunk), not after c->stream
        ac.sched = c->sched + 16 + ch;
        if ((e = cuda_ok(cudaMemsetAsync(ac.sched, 0, sizeof(int), st))) != QP_OK) return e;
        if (c->fb) {
          ac.fb_count = c->fb_ctl + 2 * (ch + qp_ctx::kPipe);
          if ((e = cuda_ok(cudaMemsetAsync(ac.fb_count, 0, 2 * sizeof(int), st))) != QP_OK) return e;
        }
      }
      c->ks.backward<<<std::min(c->grid, nb), c->ks.threads, c->L.smem, st>>>(ac);
      if ((e = cuda_ok(cudaGetLastError())) != QP_OK) return e;
      if ((e = launch_fallback(c, ac, true, ch, KP, st)) != QP_OK) return e;
      for (int f = 0; f < 6; ++f)  // per-problem gradients (a.g* is null for shared / skipped fields)
        if (gdev[f] && ghost[f] && gper[f] > 0 &&
            (e = cuda_ok(cudaMemcpyAsync(ghost[f] + (size_t)b0 * gper[f], gdev[f] + (size_t)b0 * gper[f],
                                         sizeof(float) * (size_t)nb * gper[f], cudaMemcpyDeviceToHost, st))) !=
                QP_OK)
          return e;
      if (relax_iters && (e = cuda_ok(cudaMemcpyAsync(relax_iters + b0, c->dit_ + b0, sizeof(int32_t) * nb,
                                                      cudaMemcpyDeviceToHost, st))) != QP_OK)
        return e;
      if (status && (e = cuda_ok(cudaMemcpyAsync(status + b0, c->dst_ + b0, sizeof(int32_t) * nb,
                                                 cudaMemcpyDeviceToHost, st))) != QP_OK)
        return e;
      if ((e = cuda_ok(cudaEventRecord(c->pev[ch], st))) != QP_OK) return e;
      if ((e = cuda_ok(cudaStreamWaitEvent(c->stream, c->pev[ch], 0))) != QP_OK) return e;
    }
  } else if (c->L.batched) {
    if ((e = run_batched(c, a, true)) != QP_OK) return e;
  } else if (implicit && !c->L.big && !getenv("QPB200_NO_PDL")) {
    // programmatic stream serialisation: the backward grid may start while the
    // solve grid drains (each CTA waits on done[b] for its problem), so the
    // solve's last, partly occupied wave overlaps backward work.  Both
    // launches run the same kernel (ipm_kernel), so mixed SMs share its
    // instruction cache (two separate kernels made the overlap a net loss).
    // Not on the large-N path: its per-CTA global KKT workspaces are indexed
    // by blockIdx, which a solve CTA and a backward CTA would share.
    if (c->fb && (e = cuda_ok(cudaMemsetAsync(a.fb_count, 0, 2 * sizeof(int), c->stream))) != QP_OK) return e;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(c->grid);
    lc.blockDim = dim3(c->ks.threads);
    lc.dynamicSmemBytes = c->L.smem;
    lc.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if ((e = cuda_ok(cudaLaunchKernelEx(&lc, c->ks.backward, a))) != QP_OK) return e;
    if ((e = launch_fallback(c, a, true, 0, 1, c->stream)) != QP_OK) return e;
  } else {
    if (c->fb && implicit && (e = cuda_ok(cudaMemsetAsync(a.fb_count, 0, 2 * sizeof(int), c->stream))) != QP_OK)
      return e;
    c->ks.backward<<<c->grid, c->ks.threads, c->L.smem, c->stream>>>(a);
    if ((e = cuda_ok(cudaGetLastError())) != QP_OK) return e;
    if (implicit && (e = launch_fallback(c, a, true, 0, 1, c->stream)) != QP_OK) return e;
  }
  if (shared) {
    auto osum = [&](float* out, const float* U, const float* V, const float* U2, const float* V2, int R, int Cc,
                    float scale) {
      dim3 grid((Cc + 63) / 64, (R + 63) / 64);
      qpb::outer_sum_kernel<<<grid, 256, 0, c->stream>>>(U, V, U2, V2, B, R, Cc, scale, out);
    };
    auto csum = [&](float* out, const float* U, int Cc, float scale) {
      qpb::col_sum_kernel<<<(Cc + 255) / 256, 256, 0, c->stream>>>(U, B, Cc, scale, out);
    };
    if (d.bstride_Q == 0 && oQ) osum(oQ, c->wdx, c->wx, c->wx, c->wdx, n, n, 0.5f);
    if (d.bstride_q == 0 && oq) csum(oq, c->wdx, n, 1.f);
    if (d.bstride_A == 0 && oA && m > 0) osum(oA, c->wdy, c->wx, c->wy, c->wdx, m, n, 1.f);
    if (d.bstride_b == 0 && ob && m > 0) csum(ob, c->wdy, m, -1.f);
    if (d.bstride_G == 0 && oG && p > 0) osum(oG, c->wdz, c->wx, c->wz, c->wdx, p, n, 1.f);
    if (d.bstride_h == 0 && oh && p > 0) csum(oh, c->wdz, p, -1.f);
    if ((e = cuda_ok(cudaGetLastError())) != QP_OK) return e;
  }
  if (pipe) {
    // shared-field sums (computed on c->stream after every chunk) to the host
    float* const ghost[6] = {dQ, dq, dA, db, dG, dh};
    float* const gst[6] = {c->gQ_, c->gq_, c->gA_, c->gb_, c->gG_, c->gh_};
    const int64_t bstr[6] = {d.bstride_Q, d.bstride_q, d.bstride_A, d.bstride_b, d.bstride_G, d.bstride_h};
    const size_t gper[6] = {(size_t)n * n, (size_t)n, (size_t)m * n, (size_t)m, (size_t)p * n, (size_t)p};
    for (int f = 0; f < 6; ++f)
      if (bstr[f] == 0 && ghost[f] && (e = d2h(c, ghost[f], gst[f], gper[f])) != QP_OK) return e;
    if (hsync && (e = cuda_ok(cudaStreamSynchronize(c->stream))) != QP_OK) return e;
  } else if (host) {
    if ((dQ && (e = d2h(c, dQ, c->gQ_, field_elems(d.bstride_Q, B, (size_t)n * n)))) ||
        (dq && (e = d2h(c, dq, c->gq_, field_elems(d.bstride_q, B, n)))) ||
        (dA && (e = d2h(c, dA, c->gA_, field_elems(d.bstride_A, B, (size_t)m * n)))) ||
        (db && (e = d2h(c, db, c->gb_, field_elems(d.bstride_b, B, m)))) ||
        (dG && (e = d2h(c, dG, c->gG_, field_elems(d.bstride_G, B, (size_t)p * n)))) ||
        (dh && (e = d2h(c, dh, c->gh_, field_elems(d.bstride_h, B, p)))) ||
        (relax_iters && (e = d2h(c, relax_iters, c->dit_, (size_t)B))) ||
        (status && (e = d2h(c, status, c->dst_, (size_t)B))))
      return e;
    if (hsync && (e = cuda_ok(cudaStreamSynchronize(c->stream))) != QP_OK) return e;
  }
  if (c->tl) {  // diagnostics: append {smid, start, end} of every problem (solve, then backward) to the file
    cudaStreamSynchronize(c->stream);
    std::vector<unsigned long long> h(6 * (size_t)B);
    cudaMemcpy(h.data(), c->tl, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    if (FILE* fp = fopen(getenv("QPB200_TIMELINE"), "ab")) {
      fwrite(h.data(), sizeof(unsigned long long), h.size(), fp);
      fclose(fp);
    }
  }
  return QP_OK;
}

qp_err qp_last_flops(qp_ctx* c, double* solve_flops, double* backward_flops) {
  if (!c) return QP_ERR_INVALID_ARG;
  if (cudaSetDevice(c->device) != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess) return QP_ERR_CUDA;
  const int B = c->d.batch;
  float* h = new (std::nothrow) float[B];
  if (!h) return QP_ERR_OOM;
  double sums[2] = {0.0, 0.0};
  float* src[2] = {c->flops_solve, c->flops_bwd};
  for (int w = 0; w < 2; ++w) {
    if (cudaMemcpy(h, src[w], sizeof(float) * B, cudaMemcpyDeviceToHost) != cudaSuccess) { delete[] h; return QP_ERR_CUDA; }
    for (int i = 0; i < B; ++i) sums[w] += (double)h[i];
  }
  delete[] h;
  if (solve_flops) *solve_flops = sums[0];
  if (backward_flops) *backward_flops = sums[1];
  return QP_OK;
}

qp_err qp_debug_tc_syrk(const float* G, const float* om, const float* Q, int32_t n, int32_t p, float* H,
                        void* stream) {
  if (!G || !om || !Q || !H || n < 1 || p < 1) return QP_ERR_INVALID_ARG;
  auto k = qpb::tc::debug_syrk_kernel<128>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, qpb::tc::SMEM_BYTES) != cudaSuccess)
    return QP_ERR_CUDA;
  k<<<1, 128, qpb::tc::SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(G, om, Q, n, p, H);
  return cuda_ok(cudaGetLastError());
}

qp_err qp_debug_check_guards(qp_ctx* c, int64_t* bad_words) {
  if (!c || !bad_words) return QP_ERR_INVALID_ARG;
  *bad_words = 0;
  if (!c->guard) return QP_ERR_UNSUPPORTED;
  if (cudaSetDevice(c->device) != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess) return QP_ERR_CUDA;
  std::vector<uint32_t> h(kGuard / 4);
  for (auto& g : c->guards) {
    for (int side = 0; side < 2; ++side) {
      const char* src = side == 0 ? g.first : g.first + kGuard + g.second;
      if (cudaMemcpy(h.data(), src, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return QP_ERR_CUDA;
      for (uint32_t w : h) *bad_words += (w != 0xFFFFFFFFu);
    }
  }
  return QP_OK;
}

qp_err qp_destroy(qp_ctx* c) {
  if (!c) return QP_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  free_all(c);
  for (auto& st : c->pst)
    if (st) cudaStreamDestroy(st);
  for (int l = 1; l < 4; ++l)
    if (c->bstr[l]) cudaStreamDestroy(c->bstr[l]);
  for (auto& ev : c->bev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : c->pev)
    if (ev) cudaEventDestroy(ev);
  delete c;
  return QP_OK;
}

}  // extern "C"
