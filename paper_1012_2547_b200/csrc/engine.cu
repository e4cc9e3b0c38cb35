// engine.cu -- sm_100a kernels and the C ABI of the B200 exact matcher.
//
// See scan.h for the kernel pipeline and DESIGN.md for the data layout,
// roofline and per-family byte budgets.  Reference semantics:
// pkg/src/matchbench/core.py:139-161 (all start positions, overlapping,
// ascending; m > n -> none).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <unordered_map>
#include <tuple>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "plan.h"
#include "scan.h"

#include "device_common.cuh"
#include "kernel_scan.cuh"
#include "kernel_sampled.cuh"
#include "kernel_output.cuh"
#include "kernel_mp.cuh"

using namespace mb;

// ===================================================================== C ABI

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_fail(cudaError_t e, const char* where) {
  return fail(MB_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CUDA_TRY(x)                               \
  do {                                            \
    cudaError_t e_ = (x);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)

struct mb_plan {
  PlanHost h;
  // device copy, uploaded on first use (plans are creatable without a GPU so
  // the host tables can be inspected anywhere); guarded for shared use
  mutable std::mutex mu;
  mutable uint8_t* d_buf = nullptr;  // [pattern | bloom | bucket starts | bucket entries]
  mutable PatDev* d_dev = nullptr;
  mutable PatDev dview;              // PatDev with device pointers (host copy)
  mutable int device = -1;
};

// Upload the plan to the current device once; returns the device PatDev.
static int plan_device(const mb_plan* p, const PatDev** out) {
  std::lock_guard<std::mutex> g(p->mu);
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (p->d_dev && p->device == dev) {
    *out = p->d_dev;
    return MB_OK;
  }
  if (p->d_dev) {  // used from another device: re-upload there
    cudaFree(p->d_buf);
    cudaFree(p->d_dev);
    p->d_buf = nullptr;
    p->d_dev = nullptr;
  }
  const PlanHost& h = p->h;
  const size_t pat_bytes = (size_t)((h.m + 16 + 15) & ~15LL);
  const size_t bloom_bytes = h.bloom.size() * 4;
  const size_t bs_bytes = (h.bstart.size() * 2 + 15) & ~(size_t)15;
  const size_t be_bytes = (h.bent.size() * 2 + 15) & ~(size_t)15;
  const size_t total = pat_bytes + bloom_bytes + bs_bytes + be_bytes;
  if (cudaMalloc(&p->d_buf, total) != cudaSuccess) return fail(MB_ENOMEM, "plan upload alloc");
  if (cudaMalloc(&p->d_dev, sizeof(PatDev)) != cudaSuccess) {
    cudaFree(p->d_buf);
    p->d_buf = nullptr;
    return fail(MB_ENOMEM, "plan params alloc");
  }
  std::vector<uint8_t> img(total, 0);
  memcpy(img.data(), h.pat.data(), h.m);
  if (bloom_bytes) memcpy(img.data() + pat_bytes, h.bloom.data(), bloom_bytes);
  if (!h.bstart.empty()) memcpy(img.data() + pat_bytes + bloom_bytes, h.bstart.data(), h.bstart.size() * 2);
  if (!h.bent.empty()) memcpy(img.data() + pat_bytes + bloom_bytes + bs_bytes, h.bent.data(), h.bent.size() * 2);
  CUDA_TRY(cudaMemcpy(p->d_buf, img.data(), total, cudaMemcpyHostToDevice));
  PatDev d = h.dev;
  d.bytes = p->d_buf;
  d.bloom = bloom_bytes ? reinterpret_cast<const uint32_t*>(p->d_buf + pat_bytes) : nullptr;
  d.bstart = bloom_bytes ? reinterpret_cast<const uint16_t*>(p->d_buf + pat_bytes + bloom_bytes) : nullptr;
  d.bent = bloom_bytes ? reinterpret_cast<const uint16_t*>(p->d_buf + pat_bytes + bloom_bytes + bs_bytes) : nullptr;
  CUDA_TRY(cudaMemcpy(p->d_dev, &d, sizeof(PatDev), cudaMemcpyHostToDevice));
  p->dview = d;
  p->device = dev;
  *out = p->d_dev;
  return MB_OK;
}

// what plan_pass needs of a pattern (a plan's host side, or a prepared batch's copy)
struct PatSrc {
  const uint8_t* bytes;
  int64_t m;
  int period;
};

// One batch-level pass over the text (K5; see plan_pass).
struct BatchPass {
  int kind = 0;
  int q = 0;
  int exact = 0;  // kind 2: every pattern of the pass has length q -- a gram match is an occurrence
  std::vector<uint32_t> img;                    // all chunks, each 16-byte aligned
  struct Chunk {
    int64_t off;  // word offset in img
    int B;        // log2 buckets
    int nent;     // entries
  };
  std::vector<Chunk> chunks;  // one per MP_CHUNK patterns
  int pre = 0, post = 0;                        // staged margins the verification needs
  std::vector<uint32_t> need;                   // per pattern: 0 = in the pass, 1 = per-pattern scan
  std::vector<int32_t> rep;                     // per pattern: first identical pattern of the batch (itself if none)
  std::vector<uint8_t> dcopy;                   // per duplicate: 1 = copy the representative's range afterwards
                                                // (sparse-ish outputs), 0 = expand the representative's segments
  int ndup = 0;                                 // patterns with rep[k] != k (searched once, through their rep)
  int64_t words() const { return (int64_t)img.size(); }
};

struct mb_ctx {
  int device = 0;
  int nsm = 0;
  // searches on one context share its tickets and scratch: a search on a
  // different stream than the previous one waits for that one (done_ev)
  cudaEvent_t done_ev = nullptr;
  cudaStream_t last_st = nullptr;
  bool have_last = false;
  // host entry (mb_search_batch_host): compiled plans by pattern bytes, kept
  // across calls (compile once, as the reference's harness compiles untimed)
  std::unordered_map<std::string, mb_plan*> host_plans;
  uint64_t* state = nullptr;
  int64_t state_cap = 0;
  uint16_t* counts = nullptr;
  int64_t counts_cap = 0;
  uint16_t* lists = nullptr;
  int64_t lists_cap = 0;
  uint32_t* bitmaps = nullptr;
  int64_t bitmaps_cap = 0;
  int64_t* toff = nullptr;
  int64_t toff_cap = 0;
  int64_t* seglist = nullptr;
  int64_t seglist_cap = 0;
  int64_t* qpos = nullptr;
  int64_t qpos_cap = 0;
  int32_t* rep = nullptr;  // batch pattern representatives (duplicates)
  int64_t rep_cap = 0;
  int32_t* plist = nullptr;
  int64_t plist_cap = 0;
  std::vector<int32_t> h_plist;
  uint32_t* mp_tab = nullptr;  // batch-pass tables (bloom, bucket starts, entries) per chunk
  int64_t mp_tab_cap = 0;
  uint32_t* need = nullptr;    // per-pattern scan flags of a batch pass
  int64_t need_cap = 0;
  double scratch_ok = 0;       // batch scratch bytes known to fit (skips the free-memory query)
  BatchPass pass;  // ad-hoc batches: planned per call
  int64_t mp_batches = 0;
  uint32_t epoch = 0;
  unsigned long long* ticket = nullptr;
  PatDev* d_pats = nullptr;
  int64_t pats_cap = 0;
  std::vector<PatDev> h_pats;
  // host-entry buffers
  uint8_t* d_text = nullptr;
  int64_t text_cap = 0;
  int64_t* d_out = nullptr;
  int64_t out_cap = 0;
  int64_t* d_offs = nullptr;
  int64_t offs_cap = 0;
  std::vector<mb_plan*> tmp_plans;
  cudaStream_t stream = nullptr;
  // pinned staging for the per-call uploads (batch params, MP tables, family
  // index lists): pageable cudaMemcpyAsync would block the host until the
  // stream drains.  Two arenas alternate between calls; an arena is reused
  // once the event recorded after its copies has completed.
  struct Stage {
    uint8_t* h = nullptr;
    size_t cap = 0, used = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
  } stage[2];
  int stage_i = 0;
};

// A prepared batch: device params of K plans + K5 MP tables, built once
// (mb_batch_create) and reused by every mb_find_batch_prepared call -- the
// batched analogue of the reference's compile-once / run-many split.
struct mb_batch {
  int K = 0;
  int device = 0;
  std::vector<PatDev> h_pats;
  PatDev* d_pats = nullptr;
  BatchPass pass;
  uint32_t* d_mp = nullptr;  // pass tables on the device
  int32_t* d_rep = nullptr;   // representatives (| REP_COPY) when the batch has duplicates
  uint32_t* d_need = nullptr; // per-pattern scan flags (pass / duplicates)
  // pattern bytes and periods, for re-planning the pass per sub-batch on texts
  // whose scratch does not fit the whole batch (run_batch)
  std::vector<std::vector<uint8_t>> pat_bytes;
  std::vector<PatSrc> src;
};

extern "C" {

const char* mb_last_error(void) { return g_err.c_str(); }
const char* mb_version(void) { return "matchb200 0.1.0 (sm_100a)"; }
int64_t mb_launch_count(void) { return g_launches.load(); }
int64_t mb_ctx_mp_batches(const mb_ctx* c) { return c ? c->mp_batches : 0; }

int mb_plan_create(const uint8_t* h_pattern, int64_t m, const mb_plan_opts* opts, mb_plan** out) {
  if (!out) return fail(MB_EINVAL, "null out");
  *out = nullptr;
  if (m < 1) return fail(MB_EINVAL, "pattern must have length >= 1");
  if (!h_pattern) return fail(MB_EINVAL, "null pattern");
  mb_plan* p = new mb_plan();
  std::string err;
  int rc = build_plan(h_pattern, m, opts, &p->h, &err);
  if (rc) {
    delete p;
    return fail(rc, err);
  }
  *out = p;
  return MB_OK;
}

void mb_plan_destroy(mb_plan* p) {
  if (!p) return;
  cudaFree(p->d_buf);
  cudaFree(p->d_dev);
  delete p;
}

int mb_plan_info(const mb_plan* p, mb_plan_info_t* info) {
  if (!p || !info) return fail(MB_EINVAL, "null argument");
  info->m = p->h.m;
  info->family = p->h.family;
  info->anchor = p->h.anchor;
  info->delta = p->h.dev.delta;
  info->period = p->h.period;
  info->periodic = p->h.dev.periodic;
  const bool strided = p->h.family == MB_FAM_SAMPLED || p->h.family == MB_FAM_GRAM;
  info->stride = strided ? p->h.dev.S : 0;
  info->gram = strided ? p->h.dev.q : 0;
  info->words = (p->h.family == MB_FAM_ALIGNED || p->h.family == MB_FAM_SHIFTOR) ? p->h.dev.nw : 0;
  return MB_OK;
}

int mb_plan_horspool(const mb_plan* p, int64_t* o) {
  if (!p || !o) return fail(MB_EINVAL, "null argument");
  memcpy(o, p->h.hor, sizeof(p->h.hor));
  return MB_OK;
}
int mb_plan_sunday(const mb_plan* p, int64_t* o) {
  if (!p || !o) return fail(MB_EINVAL, "null argument");
  memcpy(o, p->h.sun, sizeof(p->h.sun));
  return MB_OK;
}
int mb_plan_fwd_masks(const mb_plan* p, uint64_t* o, int64_t words) {
  if (!p || !o || words < 1) return fail(MB_EINVAL, "bad argument");
  forward_masks(p->h.pat.data(), p->h.m, o, words);
  return MB_OK;
}
int mb_plan_kmp(const mb_plan* p, int64_t* o) {
  if (!p || !o) return fail(MB_EINVAL, "null argument");
  memcpy(o, p->h.kmp.data(), sizeof(int64_t) * (p->h.m + 1));
  return MB_OK;
}
int mb_plan_gram_hash(const mb_plan* p, int q, uint32_t* o) {
  if (!p || !o) return fail(MB_EINVAL, "null argument");
  if (q != 3 && q != 5 && q != 8) return fail(MB_EINVAL, "q must be one of (3, 5, 8)");
  if (p->h.m < q) return fail(MB_EINVAL, "m < q");
  for (int64_t i = 0; i + q <= p->h.m; i++) o[i] = gram_hash(p->h.pat.data(), i, q);
  return MB_OK;
}

// Every kernel of a search prefers the maximum shared-memory carveout: the
// count kernels need it, and an SM switching carveouts between two kernels
// must drain first (a visible launch gap before each scan otherwise).
static void prefer_max_smem() {
  static std::once_flag once;
  std::call_once(once, [] {
    const void* fns[] = {(const void*)offsets_kernel<8, NT>, (const void*)offsets_kernel<16, NT>,
                         (const void*)offsets_kernel<64, NT / 2>, (const void*)expand_kernel, (const void*)fill_kernel,
                         (const void*)replicate_kernel};
    for (const void* f : fns) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaGetLastError();
  });
}

int mb_ctx_create(int device, mb_ctx** out) {
  if (!out) return fail(MB_EINVAL, "null out");
  *out = nullptr;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(MB_EINVAL, "bad device index");
  CUDA_TRY(cudaSetDevice(device));
  prefer_max_smem();
  mb_ctx* c = new mb_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&c->ticket, NTICKETS * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(c->ticket, 0, NTICKETS * sizeof(unsigned long long)) != cudaSuccess) {
    delete c;
    return fail(MB_ENOMEM, "ticket alloc");
  }
  *out = c;
  return MB_OK;
}

void mb_ctx_destroy(mb_ctx* c) {
  if (!c) return;
  for (auto& kv : c->host_plans) mb_plan_destroy(kv.second);
  cudaFree(c->state);
  cudaFree(c->counts);
  cudaFree(c->lists);
  cudaFree(c->bitmaps);
  cudaFree(c->toff);
  cudaFree(c->seglist);
  cudaFree(c->qpos);
  cudaFree(c->rep);
  cudaFree(c->plist);
  cudaFree(c->mp_tab);
  cudaFree(c->need);
  cudaFree(c->ticket);
  cudaFree(c->d_pats);
  cudaFree(c->d_text);
  cudaFree(c->d_out);
  cudaFree(c->d_offs);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->done_ev) cudaEventDestroy(c->done_ev);
  for (auto& s : c->stage) {
    if (s.ev) {
      cudaEventSynchronize(s.ev);
      cudaEventDestroy(s.ev);
    }
    cudaFreeHost(s.h);
  }
  delete c;
}

}  // extern "C"

// Occupancy (CTAs per SM) of a kernel at a dynamic smem size, cached.
static cudaError_t occupancy(const void* fn, int threads, size_t smem, int* out) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple(fn, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, threads, smem);
  if (e == cudaSuccess) cache[key] = *out;
  return e;
}

// Launch with programmatic stream serialization (PDL): the kernel may start
// before its predecessor in the stream completes and must call pdl_wait()
// before touching the predecessor's results.
// coop: the kernel passes a grid barrier (offsets_kernel's resident mode, the
// batch pass prologue) -- a cooperative launch makes the driver schedule the
// whole grid at once, so two contexts (host threads, streams) running such
// kernels concurrently cannot each hold part of the GPU and spin forever; a
// grid that could not be co-resident fails the launch instead of hanging.
template <class K, class PT>
static cudaError_t launch_ex(K kernel, int grid, int block, size_t smem, cudaStream_t st, const PT& P, bool pdl,
                             bool coop) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    na++;
  }
  if (coop) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    na++;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, P);
}
template <class K>
static cudaError_t launch_pdl(K kernel, int grid, int block, cudaStream_t st, const ScanParams& P, bool coop = false) {
  return launch_ex(kernel, grid, block, 0, st, P, true, coop);
}

// ---- pinned upload staging (see mb_ctx::stage)
static int stage_begin(mb_ctx* c) {
  c->stage_i ^= 1;
  auto& s = c->stage[c->stage_i];
  if (s.pending) {
    CUDA_TRY(cudaEventSynchronize(s.ev));
    s.pending = false;
  }
  s.used = 0;
  return MB_OK;
}
static int stage_upload(mb_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!bytes) return MB_OK;
  auto& s = c->stage[c->stage_i];
  const size_t need = s.used + ((bytes + 15) & ~(size_t)15);
  if (need > s.cap) {
    if (s.used) CUDA_TRY(cudaStreamSynchronize(st));  // this call's earlier copies still read the old arena
    cudaFreeHost(s.h);
    s.h = nullptr;
    s.cap = 0;
    s.used = 0;
    const size_t ncap = std::max<size_t>(2 * ((bytes + 15) & ~(size_t)15), 1 << 16);
    if (cudaMallocHost(&s.h, ncap) != cudaSuccess) return fail(MB_ENOMEM, "pinned staging alloc");
    s.cap = ncap;
  }
  memcpy(s.h + s.used, src, bytes);
  CUDA_TRY(cudaMemcpyAsync(dst, s.h + s.used, bytes, cudaMemcpyHostToDevice, st));
  s.used += (bytes + 15) & ~(size_t)15;
  return MB_OK;
}
static int stage_end(mb_ctx* c, cudaStream_t st) {
  auto& s = c->stage[c->stage_i];
  if (!s.used) return MB_OK;
  if (!s.ev) CUDA_TRY(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(s.ev, st));
  s.pending = true;
  return MB_OK;
}

// Stream ordering of the searches of one context (they share its tickets and
// scratch): a search on another stream than the previous one waits for it.
static int ctx_enter(mb_ctx* c, cudaStream_t st) {
  // a context's scratch, tickets and plan uploads live on its device: refuse
  // to launch from another current device (its pointers would be foreign)
  int dev = -1;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev != c->device) return fail(MB_EINVAL, "current CUDA device differs from the context's device");
  if (c->have_last && c->last_st != st) CUDA_TRY(cudaStreamWaitEvent(st, c->done_ev, 0));
  return MB_OK;
}
static int ctx_leave(mb_ctx* c, cudaStream_t st) {
  if (!c->done_ev) CUDA_TRY(cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(c->done_ev, st));
  c->last_st = st;
  c->have_last = true;
  return MB_OK;
}

// After a failed search the last kernel may not have zeroed the tickets.
static void tickets_recover(mb_ctx* c, cudaStream_t st) {
  cudaMemsetAsync(c->ticket, 0, NTICKETS * sizeof(unsigned long long), st);
}

// grow-only device scratch
template <class T>
static int grow(T** p, int64_t* cap, int64_t need, const char* what) {
  if (need <= *cap) return MB_OK;
  cudaFree(*p);
  *p = nullptr;
  int64_t ncap = std::max<int64_t>(need, 1024);
  if (cudaMalloc(p, sizeof(T) * ncap) != cudaSuccess) {
    *cap = 0;
    return fail(MB_ENOMEM, std::string("scratch alloc: ") + what);
  }
  *cap = ncap;
  return MB_OK;
}

struct SampledTag {};

// raise a kernel's dynamic smem limit once (227 KiB per CTA minus its static smem)
static cudaError_t allow_max_smem(const void* fn) {
  static std::mutex mu;
  static std::vector<const void*> done;
  std::lock_guard<std::mutex> g(mu);
  if (std::find(done.begin(), done.end(), fn) != done.end()) return cudaSuccess;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.push_back(fn);
  return e;
}

// Launch the count-producing kernel of one family group: patterns
// plist[0..gk) of the batch (indices into P.pats), ticket counter `slot`.
// *fused (optional, in/out): run the whole search as one single-wave
// scan_kernel<F, true> if every tile gets its own resident CTA; cleared when
// that does not apply (then the count kernel is launched as usual).
template <class F>
static int launch_group(mb_ctx* c, ScanParams P, const PatDev* h_pats, const int32_t* h_idx, const int32_t* d_idx,
                        int gk, int slot, cudaStream_t st, bool* fused = nullptr) {
  int pre = 0, post = 0, maxL = 0;
  int64_t maxm = 1;
  bool any_periodic = false;
  for (int i = 0; i < gk; i++) {
    const PatDev& d = h_pats[h_idx[i]];
    maxm = std::max<int64_t>(maxm, d.m);
    if (d.periodic) maxL = std::max(maxL, d.L + 1), any_periodic = true;  // +1: period-1 runs use m
    pre = std::max(pre, d.pre);
    post = std::max(post, d.post);
  }
  P.plist = d_idx;
  P.group_k = gk;
  P.group_tiles = P.ntiles * gk;
  P.ticket_slot = slot;
  P.pre = pre;
  P.post = post;
  P.pat_cap = (int)((maxm + 15) & ~15);
  P.stage_bytes = (P.pat_cap + pre + TILE + post + 127) & ~127;
  P.brk_words = any_periodic ? ((((SEG + maxL + 31) / 32) + 1 + 3) & ~3) : 0;
  if constexpr (std::is_same<F, SampledTag>::value) {
    const size_t smem_s = 8192 + 2064 + 8192 + SMP_WARPS * SMP_LIST * 4 + 16 + P.pat_cap + 16;
    static std::once_flag attr_once_s;
    cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once_s, [&] {
      attr_err = cudaFuncSetAttribute(sampled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    CUDA_TRY(attr_err);
    int per_sm_s = 0;
    CUDA_TRY(occupancy((const void*)sampled_kernel, SMP_NT, smem_s, &per_sm_s));
    if (per_sm_s < 1) return fail(MB_ECUDA, "sampled kernel does not fit on an SM");
    const int64_t wunits = (P.ntiles * NWARP + SMP_SEGS - 1) / SMP_SEGS;
    const int64_t units = ((wunits + SMP_WARPS - 1) / SMP_WARPS) * gk;
    const int64_t grid_s = std::min<int64_t>(units, (int64_t)c->nsm * per_sm_s);
    if (fused) *fused = false;
    CUDA_TRY(launch_ex(sampled_kernel, (int)grid_s, SMP_NT, smem_s, st, P, true, false));
  } else {
    auto smem_for = [&](int ns) {
      return (size_t)SM_STAGES + (size_t)ns * P.stage_bytes + NWARP * SEG_WORDS * 4 +
             (size_t)NWARP * 2 * (P.brk_words + 4) * 4 + (is_shiftor<F>::value ? NWARP * SO_WARP_WORDS * 4 : 0) +
             (is_gram<F>::value ? NWARP * GRAM_TABLE_WORDS * 4 : 0);
    };
    if (fused && *fused) {
      // one stage: each CTA stages exactly one tile
      P.nstages = 1;
      const size_t smem1 = smem_for(1);
      const void* fn = (const void*)scan_kernel<F, true>;
      CUDA_TRY(allow_max_smem(fn));
      int per_sm1 = 0;
      CUDA_TRY(occupancy(fn, NT + 32, smem1, &per_sm1));
      if (per_sm1 >= 1 && P.group_tiles <= (int64_t)c->nsm * per_sm1) {
        scan_kernel<F, true><<<(int)P.group_tiles, NT + 32, smem1, st>>>(P);
        g_launches++;
        CUDA_TRY(cudaGetLastError());
        return MB_OK;
      }
      *fused = false;
    }
    CUDA_TRY(allow_max_smem((const void*)scan_kernel<F, false>));
    // 3 stages, unless that leaves one CTA per SM where 2 stages fit two
    // (large halos: long periodic patterns keep 2 x 17 warps per SM busy)
    P.nstages = STAGES;
    size_t smem = smem_for(STAGES);
    int per_sm = 0;
    CUDA_TRY(occupancy((const void*)scan_kernel<F, false>, NT + 32, smem, &per_sm));
    if (per_sm < 2 && STAGES > 2) {
      int per_sm2 = 0;
      CUDA_TRY(occupancy((const void*)scan_kernel<F, false>, NT + 32, smem_for(2), &per_sm2));
      if (per_sm2 > per_sm) P.nstages = 2, smem = smem_for(2), per_sm = per_sm2;
    }
    if (per_sm < 1) return fail(MB_ECUDA, "scan kernel does not fit on an SM");
    const int64_t grid = std::min<int64_t>(P.group_tiles, (int64_t)c->nsm * per_sm);
    CUDA_TRY(launch_ex(scan_kernel<F, false>, (int)grid, NT + 32, smem, st, P, true, false));
  }
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

// family key: patterns sharing a key share one count-kernel launch
static int family_key(const PatDev& d) {
  if (d.family == MB_FAM_SWAR) return (int)(10 + d.m);
  if (d.family == MB_FAM_SHIFTOR) return 19 + d.nw;  // one or two symbol planes
  if (d.family == MB_FAM_ALIGNED) return d.nw == 1 && d.periodic && d.per == 1 ? 40 : 30 + d.nw;
  if (d.family == MB_FAM_WIN4 && d.nw == 2) return 50;  // even-offset windows
  if (d.family == MB_FAM_GRAM) return 60 + (d.S == 16 ? 2 : 0) + (d.q == 16 ? 1 : 0);
  return d.family;
}

static int launch_family(mb_ctx* c, const ScanParams& P, const PatDev* h_pats, const int32_t* h_idx,
                         const int32_t* d_idx, int gk, int slot, cudaStream_t st, bool* fused = nullptr) {
  const PatDev& d = h_pats[h_idx[0]];
  switch (d.family) {
    case MB_FAM_SWAR:
      switch (d.m) {
        case 1: return launch_group<FiltSWAR<1>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
        case 2: return launch_group<FiltSWAR<2>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
        case 3: return launch_group<FiltSWAR<3>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
        case 5: return launch_group<FiltSWAR<5>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
        case 6: return launch_group<FiltSWAR<6>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
        case 7: return launch_group<FiltSWAR<7>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
        case 8: return launch_group<FiltSWAR<8>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      }
      return fail(MB_EINVAL, "SWAR family needs m in 1..3 or 5..8");
    case MB_FAM_WIN4:
      if (d.nw == 2) return launch_group<FiltWIN4E>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      return launch_group<FiltWIN4>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
    case MB_FAM_ALIGNED:
      if (d.nw == 3) return launch_group<FiltALIGNED<3>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      if (d.nw == 2) return launch_group<FiltALIGNED<2>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      if (d.nw == 1 && d.periodic && d.per == 1) return launch_group<FiltRUN1>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      return launch_group<FiltALIGNED<1>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
    case MB_FAM_SAMPLED: return launch_group<SampledTag>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
    case MB_FAM_GRAM:
      if (d.S == 16 && d.q == 8) return launch_group<FiltGRAM<16, 8>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      if (d.S == 16) return launch_group<FiltGRAM<16, 16>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      if (d.q == 8) return launch_group<FiltGRAM<8, 8>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      return launch_group<FiltGRAM<8, 16>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
    case MB_FAM_SHIFTOR:
      if (d.nw == 2) return launch_group<FiltSO<2>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
      return launch_group<FiltSO<1>>(c, P, h_pats, h_idx, d_idx, gk, slot, st, fused);
  }
  return fail(MB_EINVAL, "unknown kernel family");
}

// ---- K5 batch passes: one pass over the text for a whole batch.
//
// kind 1 (aligned-word pass, mp_scan_kernel): >= 8 patterns of length >= 7
// (any family: the pass uses each plan's one-word anchor grams mpG) whose
// pooled grams hit <= 0.05 times per aligned text word; a batch of sampled
// (K3) patterns alone reads ~1/S of the text per pattern, so it takes the
// pass only from 64 patterns on.
// kind 2 (byte-offset pass, mpb_scan_kernel<q>): otherwise, >= 8 patterns of
// length >= 2 with one q-byte gram each (q = 8, 4, 3 or 2 by the shortest
// pattern), taken when every pattern expects <= 10 occurrences per 2 KiB
// segment (LIST_CAP headroom) and the pooled grams hit <= 8 times per text
// position.
// Byte probabilities p are estimated from the batch's own pattern bytes
// (patterns are drawn from the text).  Tables are built per MP_CHUNK
// patterns: bloom (64 Kbit), bucket starts, entries.

static inline uint32_t pass_hash(uint32_t lo, uint32_t hi) { return lo * 0x9E3779B1u ^ hi * 0x85EBCA77u; }
// q = 16: hash of the 4 gram words, and the fingerprint of words 2-3 kept in the entry
static inline uint32_t pass_hash16(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
  return w0 * 0x9E3779B1u ^ w1 * 0x85EBCA77u ^ w2 * 0xC2B2AE3Du ^ w3 * 0x27D4EB2Fu;
}
static inline uint32_t pass_fp16(uint32_t w2, uint32_t w3) { return w2 ^ (w3 * 0x9E3779B1u); }

template <class Ent>
static void pass_chunk(int kc, int ent_words, const Ent& ent_of, std::vector<uint32_t>& img, int* Bout, int* nout) {
  // ent_of(i, j, &hash, words[ent_words]) -> false if pattern i has no entry j
  std::vector<std::pair<uint32_t, std::vector<uint32_t>>> ents;
  for (int i = 0; i < kc; i++)
    for (int j = 0; j < 4; j++) {
      uint32_t h = 0;
      std::vector<uint32_t> w(ent_words, 0u);
      if (ent_of(i, j, &h, w.data())) ents.push_back({h, std::move(w)});
    }
  const int nent = (int)ents.size();
  int B = 4;
  while ((1 << B) < nent) B++;
  const int nb = 1 << B;
  const int bs_words = (nb + 1 + 3) & ~3;
  const size_t base = img.size();
  img.resize(base + 2048 + bs_words + (size_t)ent_words * nent, 0u);
  uint32_t* bloom = img.data() + base;
  uint32_t* bstart = bloom + 2048;
  uint32_t* out = bstart + bs_words;
  std::vector<uint32_t> cnt(nb, 0);
  for (auto& e : ents) {
    bloom[e.first >> 21] |= 1u << ((e.first >> 16) & 31);
    cnt[e.first >> (32 - B)]++;
  }
  for (int b = 0; b < nb; b++) bstart[b + 1] = bstart[b] + cnt[b];
  std::vector<uint32_t> fill(bstart, bstart + nb);
  for (auto& e : ents) {
    const uint32_t slot = fill[e.first >> (32 - B)]++;
    for (int w = 0; w < ent_words; w++) out[(size_t)ent_words * slot + w] = e.second[w];
  }
  while (img.size() % 4) img.push_back(0);
  *Bout = B;
  *nout = nent;
}

struct PatBytes {  // a pattern's bytes as plan_pass reads them
  const uint8_t* p;
  size_t n;
  const uint8_t* data() const { return p; }
  size_t size() const { return n; }
  uint8_t operator[](size_t i) const { return p[i]; }
};

static void plan_pass(const PatSrc* src, const PatDev* h_pats, int K, BatchPass* bp) {
  *bp = BatchPass();
  // identical patterns are searched once: rep[k] = first k' with the same bytes
  bp->rep.resize(K);
  {
    std::unordered_map<std::string, int> first;
    first.reserve((size_t)K * 2);
    for (int k = 0; k < K; k++) {
      const PatBytes pb{src[k].bytes, (size_t)src[k].m};
      auto ins = first.emplace(std::string(reinterpret_cast<const char*>(pb.data()), pb.size()), k);
      bp->rep[k] = ins.first->second;
      bp->ndup += ins.first->second != k;
    }
  }
  const std::vector<int32_t>& rep = bp->rep;
  double hist[256] = {0}, tot = 0;
  int64_t minm = INT64_MAX;
  for (int k = 0; k < K; k++) {
    const PatBytes pb{src[k].bytes, (size_t)src[k].m};
    const size_t lim = std::min<size_t>(pb.size(), 64);
    for (size_t i = 0; i < lim; i++) hist[pb[i]] += 1, tot += 1;
    minm = std::min<int64_t>(minm, h_pats[k].m);
  }
  double pr[256];
  for (int c = 0; c < 256; c++) pr[c] = hist[c] / tot;
  auto gp = [&](const uint8_t* g, int q) {
    double r = 1;
    for (int i = 0; i < q; i++) r *= pr[g[i]];
    return r;
  };
  // duplicates of patterns expected below 600 matches per 2 KiB segment are
  // copied from the representative's output (expansion there costs more
  // instructions per position than a copy); denser ones re-expand its
  // segments (a copy would add the source reads to a write-bound stream).
  // (256 until replicate_kernel wrote destination-line-aligned rows; config 2
  // sigma = 2, m = 2 -- 512 per segment -- copies at 0.857 ms vs 0.891 re-expanded)
  bp->dcopy.assign(K, 0);
  for (int k = 0; k < K; k++)
    if (rep[k] != k) {
      const PatBytes pb{src[k].bytes, (size_t)src[k].m};
      bp->dcopy[k] = 2048.0 * gp(pb.data(), (int)std::min<size_t>(pb.size(), 32)) < 600.0 ? 1 : 0;
    }
  if (K - bp->ndup < 8 || K > MP_CHUNK * MAX_MP_CHUNKS) return;
  // kind 1
  if (minm >= 7) {
    double rate = 0;
    bool all_sampled = true;
    for (int k = 0; k < K; k++) {
      if (rep[k] != k) continue;
      all_sampled &= h_pats[k].family == MB_FAM_SAMPLED;
      for (int j = 0; j < 4; j++) {
        uint8_t g[4];
        memcpy(g, &h_pats[k].mpG[j], 4);
        rate += gp(g, 4);
      }
    }
    if (rate <= 0.05 && (!all_sampled || K - bp->ndup >= 64)) {
      bp->kind = 1;
      bp->need.assign(K, 0u);
      int64_t pre = 0, post = 0;
      for (int k = 0; k < K; k++) {
        pre = std::max<int64_t>(pre, h_pats[k].mpa + 3);
        post = std::max<int64_t>(post, h_pats[k].m - h_pats[k].mpa + 8);
      }
      bp->pre = (int)((pre + 15) & ~15LL);
      bp->post = (int)((post + 15) & ~15LL) + 16;
      for (int k0 = 0; k0 < K; k0 += MP_CHUNK) {
        const int64_t off = (int64_t)bp->img.size();
        int B = 0, ne = 0;
        pass_chunk(std::min(MP_CHUNK, K - k0), 2,
                   [&](int i, int j, uint32_t* h, uint32_t* w) {
                     if (rep[k0 + i] != k0 + i) return false;  // searched through its representative
                     w[0] = h_pats[k0 + i].mpG[j];
                     w[1] = ((uint32_t)i << 16) | (uint32_t)(h_pats[k0 + i].mpa + j);
                     *h = w[0] * 0x9E3779B1u;  // the aligned pass hashes the word alone
                     return true;
                   },
                   bp->img, &B, &ne);
        bp->chunks.push_back({off, B, ne});
      }
      return;
    }
  }
  // kind 2: sparse patterns (<= 8 expected occurrences per 2 KiB segment, <= 2
  // if self-overlapping: a^8 clusters in a binary text) take the pass, the
  // others keep their per-pattern scan; worth it when most are sparse
  std::vector<uint32_t> need(K, 1u);
  int64_t qm = INT64_MAX, qmax = 0;
  int n_in = 0;
  // a batch of equally long short patterns (m = 2, 3, 4, 8: the gram is the
  // whole pattern, a gram match needs no verification) may be denser
  bool uniform = true;
  for (int k = 1; k < K; k++) uniform &= src[k].m == src[0].m;
  uniform &= src[0].m == 2 || src[0].m == 3 || src[0].m == 4 || src[0].m == 8;
  // (config 2, 500 patterns per 4 MiB text, limits 8 / 2 -> 16 / 8: sigma = 16, m = 2 0.334 -> 0.252 ms,
  // sigma = 2, m = 8 0.41 -> 0.375, sigma = 4, m = 4 0.377 -> 0.349; 40 / 20: sigma = 8, m = 2 0.23 -> 0.49)
  const double dens_max = uniform ? 16.0 : 8.0, dens_max_ov = uniform ? 8.0 : 2.0;
  for (int k = 0; k < K; k++) {
    const PatBytes pb{src[k].bytes, (size_t)src[k].m};
    const int64_t m = (int64_t)pb.size();
    if (rep[k] != k) {  // searched through its representative: no entry, no scan
      need[k] = 0u;
      continue;
    }
    // K3 reads ~1/S of the text on its own: a few sampled patterns keep their scans, a big
    // batch joins the pass (500 sampled scans of a 4 MiB text: 65-93 us; the pass: ~30)
    if (m < 2 || (h_pats[k].family == MB_FAM_SAMPLED && K - bp->ndup < 64)) continue;
    const double per_seg = 2048.0 * gp(pb.data(), (int)std::min<int64_t>(m, 32));
    if (per_seg > (src[k].period < m ? dens_max_ov : dens_max)) continue;
    need[k] = 0u;
    n_in++;
    qm = std::min(qm, m);
    qmax = std::max(qmax, m);
  }
  if (n_in < 8 || 2 * n_in < K - bp->ndup) return;
  int q = qm >= 8 ? 8 : qm >= 4 ? 4 : (int)qm;
  if (q == 8 && qm >= 16) {
    // 8-byte grams of small alphabets hit at most text positions (sigma = 2:
    // 8 bits each, 500 patterns cover all 256 values): 16-byte grams when the
    // 8-byte pool would hit more than 0.05 times per position
    double pool8 = 0;
    for (int k = 0; k < K; k++)
      if (!need[k] && rep[k] == k) {
        double best = 1;
        const PatBytes pb{src[k].bytes, (size_t)src[k].m};
        for (int64_t a = 0; a + 8 <= (int64_t)pb.size(); a++) best = std::min(best, gp(pb.data() + a, 8));
        pool8 += best;
      }
    if (pool8 > 0.05) q = 16;
  }
  std::vector<int32_t> anchor(K, 0);
  std::unordered_map<std::string, int> used;  // gram value -> patterns already anchored on it
  double pooled = 0;
  for (int k = 0; k < K; k++) {
    if (need[k] || rep[k] != k) continue;
    const PatBytes pb{src[k].bytes, (size_t)src[k].m};
    const int64_t m = (int64_t)pb.size();
    // rarest window, spread over distinct gram values (a value shared by many
    // patterns makes every text hit on it walk all of them)
    int best = 0;
    double bcost = 1e300, bpr = 0;
    std::string bval;
    for (int64_t a = 0; a + q <= m; a++) {
      const std::string v(reinterpret_cast<const char*>(pb.data() + a), q);
      const double r = gp(pb.data() + a, q);
      auto it = used.find(v);
      const double cost = r * (1 + (it == used.end() ? 0 : it->second));
      if (cost < bcost * (1 - 1e-12)) bcost = cost, bpr = r, best = (int)a, bval = v;
    }
    anchor[k] = best;
    used[bval]++;
    pooled += bpr;
  }
  if (pooled > 8.0) return;
  bp->kind = 2;
  bp->q = q;
  bp->exact = (q != 16 && qm == q && qmax == q) ? 1 : 0;
  for (int k = 0; k < K && bp->exact; k++)
    if (!need[k] && rep[k] == k && (anchor[k] != 0 || h_pats[k].delta < 0 || h_pats[k].delta > 0xFFFF)) bp->exact = 0;
  const bool exact = bp->exact != 0;
  bp->need = need;
  int64_t pre = 0, post = 0;
  for (int k = 0; k < K; k++) {
    if (need[k] || rep[k] != k) continue;
    pre = std::max<int64_t>(pre, anchor[k]);
    post = std::max<int64_t>(post, h_pats[k].m - anchor[k] + 8);
  }
  bp->pre = (int)((pre + 15) & ~15LL);
  bp->post = (int)((std::max<int64_t>(post, q == 16 ? 36 : 24) + 15) & ~15LL) + 16;
  for (int k0 = 0; k0 < K; k0 += MP_CHUNK) {
    const int64_t off = (int64_t)bp->img.size();
    int B = 0, ne = 0;
    pass_chunk(std::min(MP_CHUNK, K - k0), 4,
               [&](int i, int j, uint32_t* h, uint32_t* w) {
                 if (j || need[k0 + i] || rep[k0 + i] != k0 + i) return false;  // one gram per pattern in the pass
                 const PatBytes pb{src[k0 + i].bytes, (size_t)src[k0 + i].m};
                 uint8_t g[16] = {0};
                 memcpy(g, pb.data() + anchor[k0 + i], q);
                 uint32_t gw[4];
                 memcpy(gw, g, 16);
                 w[0] = gw[0];
                 w[1] = gw[1];
                 // (exact pass: the anchor is 0 and the slot carries the family's bitmap shift)
                 w[2] = ((uint32_t)i << 16) | (uint32_t)(exact ? h_pats[k0 + i].delta : anchor[k0 + i]);
                 w[3] = q == 16 ? pass_fp16(gw[2], gw[3]) : 0u;
                 *h = q == 16 ? pass_hash16(gw[0], gw[1], gw[2], gw[3]) : pass_hash(w[0], w[1]);
                 return true;
               },
               bp->img, &B, &ne);
    bp->chunks.push_back({off, B, ne});
  }
}

// One search (K = 1) or batch: per family group one count kernel (or, for a
// selective batch of anchor-filter patterns, one MP pass over the text), then
// one offsets and one expand launch over all K patterns' segments, so the
// output is CSR in the caller's pattern order whatever the family mix.
// Batch-only inputs of run_search (a single search passes none).
struct SubBatch {
  const BatchPass* bp = nullptr;     // batch-pass plan (null / kind 0: no pass)
  const uint32_t* d_tab = nullptr;   // its tables on the device
  int chunk0 = 0;                    // first pass-table chunk of this sub-batch
  // host, this sub-batch's indices (null = identity / scan all): each
  // pattern's representative (identical patterns are searched once: offsets
  // and expand read the representative's segments for the duplicate's CSR
  // range, or replicate_kernel copies its output when | REP_COPY) and the
  // per-pattern scan flags (0: covered by the batch pass or by its
  // representative -- the count kernels skip its tiles)
  const int32_t* h_rep = nullptr;
  const uint32_t* h_need = nullptr;
  int64_t* csr0 = nullptr;           // the CSR's leading entry, zeroed by the search
  const int32_t* d_rep = nullptr;    // prepared batch: h_rep already resident on the device
  const uint32_t* d_need = nullptr;  // prepared batch: h_need already resident on the device
};

static int run_search(mb_ctx* c, const PatDev* d_pats, const PatDev* h_pats, int K, const uint8_t* d_text,
                      int64_t n, int64_t* d_out, int64_t cap, int64_t* offsets_plus1, cudaStream_t st,
                      const int64_t* out_base = nullptr, const SubBatch& sb = SubBatch()) {
  const BatchPass* bp = sb.bp;
  const uint32_t* d_tab = sb.d_tab;
  const int chunk0 = sb.chunk0;
  const int32_t* h_rep = sb.h_rep;
  const uint32_t* h_need = sb.h_need;
  int64_t* csr0 = sb.csr0;
  const int32_t* d_rep_pre = sb.d_rep;
  const uint32_t* d_need_pre = sb.d_need;
  ScanParams P;
  memset(&P, 0, sizeof(P));
  const uintptr_t addr = (uintptr_t)d_text;
  P.text = (const uint8_t*)(addr & ~(uintptr_t)15);
  P.off = (int64_t)(addr & 15);
  P.n = n;
  P.nv16 = (P.off + n + 15) & ~(int64_t)15;
  int64_t nbits = 0;
  for (int k = 0; k < K; k++)
    if (h_pats[k].m <= n) nbits = std::max<int64_t>(nbits, P.off + h_pats[k].delta + n - h_pats[k].m + 1);
  if (nbits == 0 && csr0) CUDA_TRY(cudaMemsetAsync(csr0, 0, sizeof(int64_t), st));
  if (nbits == 0) {  // every pattern longer than the text: no output, offsets stay at the base
    if (out_base) {
      fill_kernel<<<(K + 255) / 256, 256, 0, st>>>(offsets_plus1, out_base, K);
      g_launches++;
      CUDA_TRY(cudaGetLastError());
    } else {
      CUDA_TRY(cudaMemsetAsync(offsets_plus1, 0, sizeof(int64_t) * K, st));
    }
    return MB_OK;
  }
  P.ntiles = (nbits + TILE - 1) / TILE;
  P.total_tiles = P.ntiles * K;
  P.pats = d_pats;
  P.K = K;
  const int64_t T = P.total_tiles * NWARP;  // segments
  // offsets_kernel chunk: the largest of NT*{32,16,8} counts that still gives
  // >= 2 chunks per SM (short texts otherwise leave the scan on a few SMs)
  const int scan_per = T >= (int64_t)NT * 32 * 2 * c->nsm ? 32 : T >= (int64_t)NT * 16 * 2 * c->nsm ? 16 : 8;
  const int64_t chunk = (int64_t)NT * scan_per;
  const int64_t nchunks = (T + chunk - 1) / chunk;
  int rc;
  // whole chunks (offsets_kernel reads 16-byte vectors) + 2 slots for the MP overflow flag
  if ((rc = grow(&c->counts, &c->counts_cap, nchunks * chunk + 8, "counts"))) return rc;
  if ((rc = grow(&c->lists, &c->lists_cap, T * LIST_CAP, "lists"))) return rc;
  if ((rc = grow(&c->bitmaps, &c->bitmaps_cap, T * SEG_WORDS, "bitmaps"))) return rc;
  if ((rc = grow(&c->toff, &c->toff_cap, T, "tile offsets"))) return rc;
  if ((rc = grow(&c->seglist, &c->seglist_cap, T, "expand queue"))) return rc;
  if ((rc = grow(&c->qpos, &c->qpos_cap, T, "expand queue positions"))) return rc;
  // look-back flags: per offsets chunk, or per tile of a fused single-wave search
  const int64_t nstate = std::max<int64_t>(nchunks, K == 1 ? std::min<int64_t>(P.total_tiles, 4 * (int64_t)c->nsm) : 0);
  if (nstate > c->state_cap || c->epoch >= (1u << 24) - 4) {
    if ((rc = grow(&c->state, &c->state_cap, nstate, "look-back state"))) return rc;
    CUDA_TRY(cudaMemsetAsync(c->state, 0, sizeof(uint64_t) * c->state_cap, st));
    // the epoch parity picks the expand-queue slot: restart it with clean tickets
    CUDA_TRY(cudaMemsetAsync(c->ticket, 0, NTICKETS * sizeof(unsigned long long), st));
    c->epoch = 0;
  }
  P.counts = c->counts;
  P.lists = c->lists;
  P.bitmaps = c->bitmaps;
  P.toff = c->toff;
  P.seglist = c->seglist;
  P.qpos = c->qpos;
  int ndup = 0;  // duplicates in this (sub-)batch
  if (h_rep) {
    for (int k = 0; k < K; k++) ndup += (h_rep[k] & REP_COPY) != 0;  // duplicates filled by replicate_kernel
    if (d_rep_pre) {  // prepared batch: resident on the device
      P.rep = d_rep_pre;
    } else {
      if ((rc = grow(&c->rep, &c->rep_cap, K, "pattern representatives"))) return rc;
      if ((rc = stage_upload(c, c->rep, h_rep, sizeof(int32_t) * K, st))) return rc;
      P.rep = c->rep;
    }
  }
  P.state = c->state;
  P.ticket = c->ticket;
  P.out = d_out;
  P.cap = d_out ? cap : 0;
  P.offsets_plus1 = offsets_plus1;
  P.out_base = out_base;
  P.csr0 = csr0;

  // one epoch per search: look-back flags of older searches never match, and
  // its parity picks the expand-queue ticket slot (consecutive searches alternate)
  P.epoch = ++c->epoch;
  auto finish = [&](bool unsorted) -> int {
    P.unsorted_lists = unsorted ? 1 : 0;
    // programmatic dependent launches: offsets/expand CTAs are scheduled as the
    // previous grid drains and wait in-kernel (griddepcontrol.wait) for its
    // results -- the launch gap and the scan's tail overlap
    P.dense_slot = (P.epoch & 1) ? TICKET_DENSE_ODD : TICKET_DENSE;
    // chunk = NT * scan_per counts; the largest chunks run as 256-thread CTAs
    // x 64 counts (4 CTAs per SM, so 16 GiB's 512 chunks stay co-resident)
    // co-resident grids of more than 32 chunks: grid barrier (a cooperative launch, which
    // cannot start before its predecessor has drained: ~3 us after the scan's last CTA).
    // Up to 32 chunks (single searches up to ~256 MiB) the ticket-ordered look-back is one
    // round trip and the kernel stays a plain dependent launch, resident while the scan drains
    P.offs_resident = (nchunks > 32 && nchunks <= (int64_t)c->nsm * (scan_per == 32 ? 4 : 2)) ? 1 : 0;  // __launch_bounds__
    const bool coop = P.offs_resident != 0;  // grid barrier: cooperative launch (see launch_ex)
    if (scan_per == 32)
      CUDA_TRY(launch_pdl(offsets_kernel<64, NT / 2>, (int)nchunks, NT / 2, st, P, coop));
    else if (scan_per == 16)
      CUDA_TRY(launch_pdl(offsets_kernel<16, NT>, (int)nchunks, NT, st, P, coop));
    else
      CUDA_TRY(launch_pdl(offsets_kernel<8, NT>, (int)nchunks, NT, st, P, coop));
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    if (d_out && cap > 0) {
      // one resident wave at most: the CTAs are scheduled while offsets_kernel
      // runs (it triggers its dependents at entry) and loop over the queue
      int exp_per_sm = 0;
      CUDA_TRY(occupancy((const void*)expand_kernel, EXP_WARPS * 32, 0, &exp_per_sm));
      // CTAs per SM capped (MB_EXP_CTAS, tuning): fewer concurrently advancing 16 KB
      // output regions keep more of their DRAM pages open (tools/probe_expand_pattern.cu)
      static const int exp_cap = [] { const char* e = getenv("MB_EXP_CTAS"); return e ? atoi(e) : 8; }();
      const int64_t eg = std::min<int64_t>((T + EXP_WARPS - 1) / EXP_WARPS,
                                           (int64_t)c->nsm * std::max(std::min(exp_per_sm, exp_cap), 1));
      CUDA_TRY(launch_pdl(expand_kernel, (int)eg, EXP_WARPS * 32, st, P));
      g_launches++;
      CUDA_TRY(cudaGetLastError());
      if (ndup) {  // duplicates marked REP_COPY: copy the representatives' ranges
        CUDA_TRY(launch_pdl(replicate_kernel, K > REPL_MAXK ? (int)std::min<int64_t>(K, (int64_t)c->nsm * 4) : c->nsm * 4, 512, st, P));
        g_launches++;
        CUDA_TRY(cudaGetLastError());
      }
    }
    return MB_OK;
  };

  bool mp_used = false;
  if (bp && bp->kind && d_tab) {
    MPParams M;
    memset(&M, 0, sizeof(M));
    M.text = P.text;
    M.off = P.off;
    M.n = n;
    M.nv16 = P.nv16;
    M.ntiles_text = (P.nv16 + TILE - 1) / TILE;
    M.ntiles = P.ntiles;
    M.pre = bp->pre;
    M.post = bp->post;
    M.stage_bytes = (M.pre + TILE + M.post + 127) & ~127;
    M.pats = d_pats;
    M.counts = c->counts;
    M.lists = c->lists;
    M.overflow = reinterpret_cast<unsigned int*>(c->counts + T);  // 4 spare bytes after the counts
    // per-pattern scan flags (patterns left out of the pass start at 1): from
    // the prepared batch's device copy inside the pass prologue, else uploaded;
    // the prologue also zeroes the counts (the pass counts with atomics)
    if ((rc = grow(&c->need, &c->need_cap, K, "pass flags"))) return rc;
    if (!d_need_pre && (rc = stage_upload(c, c->need, h_need, sizeof(uint32_t) * K, st))) return rc;
    M.need = c->need;
    M.need_src = d_need_pre;
    M.need_k = K;
    M.bar = c->ticket + TICKET_MPBAR;
    // tickets are zero: the previous search's last kernel reset them
    const void* fn = bp->kind == 1 ? (const void*)mp_scan_kernel
                     : bp->q == 16 ? (const void*)mpb_scan_kernel<16>
                     : bp->q == 8  ? (const void*)mpb_scan_kernel<8>
                     : bp->q == 4  ? (const void*)mpb_scan_kernel<4>
                     : bp->q == 3  ? (const void*)mpb_scan_kernel<3>
                                   : (const void*)mpb_scan_kernel<2>;
    {
      static std::mutex mu_mp;
      static std::vector<const void*> attr_done;
      std::lock_guard<std::mutex> g(mu_mp);
      if (std::find(attr_done.begin(), attr_done.end(), fn) == attr_done.end()) {
        CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_done.push_back(fn);
      }
    }
    const int ent_words = bp->kind == 1 ? 2 : 4;
    for (int k0 = 0, ci = chunk0; k0 < K; k0 += MP_CHUNK, ci++) {
      const int B = bp->chunks[ci].B;
      const int bs_words = ((1 << B) + 1 + 3) & ~3;
      M.bloom = d_tab + bp->chunks[ci].off;
      M.bstart = M.bloom + 2048;
      M.ents = reinterpret_cast<const uint2*>(M.bstart + bs_words);
      M.ents4 = reinterpret_cast<const uint4*>(M.bstart + bs_words);
      M.B = B;
      M.nents = bp->chunks[ci].nent;
      M.kbase = k0;
      M.exact_m = (bp->kind == 2 && bp->exact) ? bp->q : 0;
      M.exact_local = 0;
      if (M.exact_m) {  // every pass pattern of this chunk at bitmap shift 0 (SWAR, K2, m = 4 windows at anchor 0)
        M.exact_local = 1;
        for (int k = k0; k < std::min(K, k0 + MP_CHUNK); k++)
          if (!h_need[k] && (!h_rep || (h_rep[k] & ~REP_COPY) == k) && h_pats[k].delta != 0) M.exact_local = 0;
      }
      M.ticket = c->ticket + TICKET_MP0 + (ci - chunk0);
      M.zero_n = k0 == 0 ? T + 2 : 0;  // the first launch's prologue (its grid is co-resident)
      auto smem_for = [&](int ns) {
        return (size_t)SM_STAGES + (size_t)ns * M.stage_bytes + 8192 + 4 * bs_words + (size_t)4 * ent_words * M.nents +
               (M.exact_local ? (size_t)NWARP * MP_CHUNK * 2 + 16 : 0);
      };
      // 3 stages, or for the aligned pass 2 where that keeps two CTAs per SM
      // (big tables / halos; measured 55 -> 40 us on config 3, m = 16).  The
      // byte-offset pass is bound by its smem bloom lookups: a second CTA
      // does not help it and the shallower ring hurts (sigma = 2: +18%).
      M.nstages = STAGES;
      size_t smem = smem_for(STAGES);
      int per_sm = 0;
      CUDA_TRY(occupancy(fn, NT + 32, smem, &per_sm));
      if (bp->kind == 1 && per_sm < 2 && STAGES > 2) {
        int per_sm2 = 0;
        CUDA_TRY(occupancy(fn, NT + 32, smem_for(2), &per_sm2));
        if (per_sm2 > per_sm) M.nstages = 2, smem = smem_for(2), per_sm = per_sm2;
      }
      if (per_sm < 1) return fail(MB_ECUDA, "batched pass kernel does not fit on an SM");
      const int grid = (int)std::min<int64_t>(M.ntiles_text, (int64_t)c->nsm * per_sm);
      // the first launch's prologue ends in a grid barrier: cooperative (see launch_ex)
      const bool coop = M.zero_n > 0;
      cudaError_t le;
      if (bp->kind == 1)
        le = launch_ex(mp_scan_kernel, grid, NT + 32, smem, st, M, false, coop);
      else if (bp->q == 16)
        le = launch_ex(mpb_scan_kernel<16>, grid, NT + 32, smem, st, M, false, coop);
      else if (bp->q == 8)
        le = launch_ex(mpb_scan_kernel<8>, grid, NT + 32, smem, st, M, false, coop);
      else if (bp->q == 4)
        le = launch_ex(mpb_scan_kernel<4>, grid, NT + 32, smem, st, M, false, coop);
      else if (bp->q == 3)
        le = launch_ex(mpb_scan_kernel<3>, grid, NT + 32, smem, st, M, false, coop);
      else
        le = launch_ex(mpb_scan_kernel<2>, grid, NT + 32, smem, st, M, false, coop);
      CUDA_TRY(le);
      g_launches++;
      CUDA_TRY(cudaGetLastError());
    }
    // fallback without a host round trip: the per-pattern scan below runs only if
    // a segment overflowed (kernels read the flag and exit otherwise); lists are
    // sorted on expand either way (harmless for the already-sorted fallback lists)
    P.run_if = M.overflow;
    P.need = c->need;
    mp_used = true;
    c->mp_batches++;
  }
  // tickets are zero here: ctx creation, or the previous search's last kernel reset them
  if (K == 1 && !mp_used) {
    // one pattern: the whole search as one single-wave launch when every tile
    // fits a resident CTA (texts up to ~9 MiB), else the count kernel + finish
    bool fused = true;
    const int32_t idx0 = 0;
    if ((rc = launch_family(c, P, h_pats, &idx0, nullptr, 1, 0, st, &fused))) return rc;
    return fused ? MB_OK : finish(false);
  }
  // count kernels, one launch per family key (stable groups): the patterns
  // that need a scan (all; or those the batch pass left out, and the
  // representatives of duplicates) unconditionally; with a batch pass, its
  // own patterns once more behind the overflow flag -- those launches exit at
  // once unless a pass segment overflowed, and then scan only the patterns
  // whose flag the pass set
  const uint32_t* run_if_pass = P.run_if;
  std::vector<int> keys;
  std::vector<std::vector<int32_t>> groups;
  std::vector<char> gated;
  auto add = [&](int k, bool gate) {
    const int key = family_key(h_pats[k]) * 2 + (gate ? 1 : 0);
    size_t g = 0;
    while (g < keys.size() && keys[g] != key) g++;
    if (g == keys.size()) {
      keys.push_back(key);
      groups.emplace_back();
      gated.push_back(gate ? 1 : 0);
    }
    groups[g].push_back(k);
  };
  int nlisted = 0;
  for (int k = 0; k < K; k++)
    if (!h_need || h_need[k]) add(k, false), nlisted++;
  if (mp_used)
    for (int k = 0; k < K; k++)
      if (!h_need[k] && (!h_rep || h_rep[k] == k)) add(k, true), nlisted++;  // (h_rep[k] == k: no flag)
  // at most NFAMILY_KEYS keys, each once ungated and once gated: always fits
  if ((int)groups.size() > MAX_GROUPS) return fail(MB_ECUDA, "internal: more family groups than ticket slots");
  const bool identity = groups.size() == 1 && nlisted == K;  // all patterns in order: no index list needed
  if (!identity && nlisted) {
    if ((rc = grow(&c->plist, &c->plist_cap, nlisted, "family index lists"))) return rc;
    c->h_plist.clear();
    for (auto& g : groups) c->h_plist.insert(c->h_plist.end(), g.begin(), g.end());
    if ((rc = stage_upload(c, c->plist, c->h_plist.data(), sizeof(int32_t) * nlisted, st))) return rc;
  }
  int base = 0;
  for (size_t g = 0; g < groups.size(); g++) {
    ScanParams Pg = P;
    Pg.run_if = gated[g] ? run_if_pass : nullptr;
    Pg.need = gated[g] ? P.need : nullptr;
    if ((rc = launch_family(c, Pg, h_pats, groups[g].data(), identity ? nullptr : c->plist + base,
                            (int)groups[g].size(), (int)g, st)))
      return rc;
    base += (int)groups[g].size();
  }
  return finish(mp_used);
}

extern "C" {

int mb_find(mb_ctx* c, const mb_plan* p, const uint8_t* d_text, int64_t n, int64_t* d_out, int64_t cap,
            int64_t* d_count, void* stream) {
  if (!c || !p || !d_count) return fail(MB_EINVAL, "null argument");
  if (n < 0 || cap < 0) return fail(MB_EINVAL, "negative size");
  if (n > 0 && !d_text) return fail(MB_EINVAL, "null text");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ctx_enter(c, st);
  if (rc) return rc;
  if (p->h.m > n) {
    CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(int64_t), st));
    return ctx_leave(c, st);
  }
  const PatDev* dd = nullptr;
  if ((rc = plan_device(p, &dd))) return rc;
  if ((rc = stage_begin(c))) return rc;
  rc = run_search(c, dd, &p->dview, 1, d_text, n, d_out, cap, d_count, st);
  if (rc) tickets_recover(c, st);
  const int rc2 = stage_end(c, st);
  const int rc3 = ctx_leave(c, st);
  return rc ? rc : rc2 ? rc2 : rc3;
}

// Run a batch whose params are on the device as sub-batches under the scratch
// budget (~346 B per 2 KiB segment per pattern: counts, list, bitmap, offset, position,
// queue; a third of free memory, <= 16 GiB), chained through d_offsets.
static int run_batch(mb_ctx* c, const PatDev* d_pats, const PatDev* h_pats, int K, const uint8_t* d_text, int64_t n,
                     int64_t* d_out, int64_t cap, int64_t* d_offsets, cudaStream_t st, const BatchPass* bp,
                     const uint32_t* d_tab, const PatSrc* src, const int32_t* d_rep_pre = nullptr,
                     const uint32_t* d_need_pre = nullptr) {
  const double per_pattern = (double)((n + 2 * MB_MAX_M + TILE) / TILE + 1) * NWARP * 346.0;
  // batches needing <= 1 GiB of scratch, or no more than a previous call
  // already got, skip the memory query (cudaMemGetInfo costs up to ms)
  double budget = std::max(1.0 * (1ULL << 30), c->scratch_ok);
  if (const char* env = getenv("MB_SCRATCH_BUDGET")) {
    budget = atof(env);  // tests force sub-batching
  } else if (per_pattern * K > budget) {
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    budget = std::max(budget, std::min<double>((double)free_b / 3.0, 16.0 * (1ULL << 30)));
    c->scratch_ok = std::max(c->scratch_ok, std::min(budget, per_pattern * K));
  }
  int kc = (int)std::max<double>(1.0, std::min<double>((double)K, budget / per_pattern));
  if (kc < K && kc >= MP_CHUNK) kc -= kc % MP_CHUNK;  // keep the pass tables' chunks aligned to sub-batches
  std::vector<int32_t> lrep;
  std::vector<uint32_t> lneed;
  if (kc < K && src) {
    // The text is too large for the whole batch's scratch: every sub-batch is
    // planned on its own (duplicates and the batch pass among its patterns),
    // so it still reads the text once -- not once per pattern.  Host planning
    // and a table upload per sub-batch: negligible against GiB-sized scans.
    for (int k0 = 0; k0 < K; k0 += kc) {
      const int kk = std::min(kc, K - k0);
      BatchPass sp;
      plan_pass(src + k0, h_pats + k0, kk, &sp);
      const bool dups = sp.ndup > 0, whole = sp.kind != 0;
      lrep.resize(kk);
      lneed.resize(kk);
      for (int i = 0; i < kk; i++) {
        lrep[i] = sp.rep[i];
        if (lrep[i] != i && sp.dcopy[i]) lrep[i] |= REP_COPY;
        lneed[i] = whole ? sp.need[i] : (sp.rep[i] == i ? 1u : 0u);
      }
      int rc;
      if (whole) {
        if ((rc = grow(&c->mp_tab, &c->mp_tab_cap, sp.words(), "batch pass tables"))) return rc;
        if ((rc = stage_upload(c, c->mp_tab, sp.img.data(), sizeof(uint32_t) * sp.img.size(), st))) return rc;
      }
      SubBatch sb;
      sb.bp = whole ? &sp : nullptr;
      sb.d_tab = whole ? c->mp_tab : nullptr;
      sb.chunk0 = 0;
      sb.h_rep = dups ? lrep.data() : nullptr;
      sb.h_need = (dups || whole) ? lneed.data() : nullptr;
      sb.csr0 = k0 == 0 ? d_offsets : nullptr;
      rc = run_search(c, d_pats + k0, h_pats + k0, kk, d_text, n, d_out, cap, d_offsets + 1 + k0, st,
                      k0 ? d_offsets + k0 : nullptr, sb);
      if (rc) return rc;
    }
    return MB_OK;
  }
  for (int k0 = 0; k0 < K; k0 += kc) {
    const int kk = std::min(kc, K - k0);
    // the pass runs on sub-batches made of whole table chunks
    const bool whole = bp && bp->kind && (k0 % MP_CHUNK) == 0 && (kk % MP_CHUNK == 0 || k0 + kk == K);
    // representatives inside this sub-batch; a duplicate whose representative
    // is in another sub-batch is scanned here (it has no pass-table entry)
    const bool dups = bp && bp->ndup > 0 && (int)bp->rep.size() == K;
    if (dups || whole) {
      lrep.resize(kk);
      lneed.resize(kk);
      for (int i = 0; i < kk; i++) {
        const int r = dups ? bp->rep[k0 + i] : k0 + i;
        lrep[i] = r >= k0 ? r - k0 : i;
        if (lrep[i] != i && bp->dcopy[k0 + i]) lrep[i] |= REP_COPY;  // copy the representative's range
        const bool orphan = r != k0 + i && r < k0;
        lneed[i] = whole ? (orphan ? 1u : bp->need[k0 + i]) : (lrep[i] == i ? 1u : 0u);
      }
    }
    // the whole batch in one go: a prepared batch's device-resident flags
    const bool all = k0 == 0 && kk == K;
    SubBatch sb;
    sb.bp = whole ? bp : nullptr;
    sb.d_tab = whole ? d_tab : nullptr;
    sb.chunk0 = k0 / MP_CHUNK;
    sb.h_rep = dups ? lrep.data() : nullptr;
    sb.h_need = (dups || whole) ? lneed.data() : nullptr;
    sb.csr0 = k0 == 0 ? d_offsets : nullptr;
    sb.d_rep = all ? d_rep_pre : nullptr;
    sb.d_need = all ? d_need_pre : nullptr;
    int rc = run_search(c, d_pats + k0, h_pats + k0, kk, d_text, n, d_out, cap, d_offsets + 1 + k0, st,
                        k0 ? d_offsets + k0 : nullptr, sb);
    if (rc) return rc;
  }
  return MB_OK;
}

int mb_find_batch(mb_ctx* c, const mb_plan* const* plans, int K, const uint8_t* d_text, int64_t n,
                  int64_t* d_out, int64_t cap, int64_t* d_offsets, void* stream) {
  if (!c || !plans || K < 1 || !d_offsets) return fail(MB_EINVAL, "bad argument");
  if (n < 0 || cap < 0) return fail(MB_EINVAL, "negative size");
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = ctx_enter(c, st))) return rc;
  c->h_pats.resize(K);
  for (int k = 0; k < K; k++) {
    if (!plans[k]) return fail(MB_EINVAL, "null plan in batch");
    const PatDev* dd = nullptr;
    int rc = plan_device(plans[k], &dd);
    if (rc) return rc;
    c->h_pats[k] = plans[k]->dview;
  }
  if ((rc = grow(&c->d_pats, &c->pats_cap, K, "batch params"))) return rc;
  if ((rc = stage_begin(c))) return rc;
  if ((rc = stage_upload(c, c->d_pats, c->h_pats.data(), sizeof(PatDev) * K, st))) return rc;
  std::vector<PatSrc> src(K);
  for (int k = 0; k < K; k++) src[k] = PatSrc{plans[k]->h.pat.data(), plans[k]->h.m, plans[k]->h.period};
  plan_pass(src.data(), c->h_pats.data(), K, &c->pass);
  if (c->pass.kind) {
    if ((rc = grow(&c->mp_tab, &c->mp_tab_cap, c->pass.words(), "batch pass tables"))) return rc;
    if ((rc = stage_upload(c, c->mp_tab, c->pass.img.data(), sizeof(uint32_t) * c->pass.img.size(), st))) return rc;
  }
  rc = run_batch(c, c->d_pats, c->h_pats.data(), K, d_text, n, d_out, cap, d_offsets, st, &c->pass, c->mp_tab,
                 src.data());
  if (rc) tickets_recover(c, st);
  const int rc2 = stage_end(c, st);
  const int rc3 = ctx_leave(c, st);
  return rc ? rc : rc2 ? rc2 : rc3;
}

int mb_batch_create(const mb_plan* const* plans, int K, mb_batch** out) {
  if (!out || !plans || K < 1) return fail(MB_EINVAL, "bad argument");
  *out = nullptr;
  mb_batch* b = new mb_batch();
  b->K = K;
  b->h_pats.resize(K);
  for (int k = 0; k < K; k++) {
    const PatDev* dd = nullptr;
    int rc = plans[k] ? plan_device(plans[k], &dd) : fail(MB_EINVAL, "null plan in batch");
    if (rc) {
      delete b;
      return rc;
    }
    b->h_pats[k] = plans[k]->dview;
  }
  cudaGetDevice(&b->device);
  b->pat_bytes.resize(K);
  b->src.resize(K);
  for (int k = 0; k < K; k++) {
    b->pat_bytes[k] = plans[k]->h.pat;
    b->src[k] = PatSrc{b->pat_bytes[k].data(), plans[k]->h.m, plans[k]->h.period};
  }
  plan_pass(b->src.data(), b->h_pats.data(), K, &b->pass);
  const BatchPass& bp = b->pass;
  const std::vector<uint32_t>& img = bp.img;
  // the whole batch's representative / scan-flag arrays (run_batch's sub-batch
  // arrays for one sub-batch), resident so a call uploads nothing
  const bool dups = bp.ndup > 0, whole = bp.kind != 0;
  std::vector<int32_t> lrep(K);
  std::vector<uint32_t> lneed(K);
  for (int k = 0; k < K; k++) {
    lrep[k] = bp.rep[k];
    if (lrep[k] != k && bp.dcopy[k]) lrep[k] |= REP_COPY;
    lneed[k] = whole ? bp.need[k] : (bp.rep[k] == k ? 1u : 0u);
  }
  cudaError_t e = cudaMalloc(&b->d_pats, sizeof(PatDev) * K);
  if (e == cudaSuccess && !img.empty()) e = cudaMalloc(&b->d_mp, sizeof(uint32_t) * img.size());
  if (e == cudaSuccess && dups) e = cudaMalloc(&b->d_rep, sizeof(int32_t) * K);
  if (e == cudaSuccess && (dups || whole)) e = cudaMalloc(&b->d_need, sizeof(uint32_t) * K);
  if (e == cudaSuccess) e = cudaMemcpy(b->d_pats, b->h_pats.data(), sizeof(PatDev) * K, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !img.empty())
    e = cudaMemcpy(b->d_mp, img.data(), sizeof(uint32_t) * img.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && b->d_rep) e = cudaMemcpy(b->d_rep, lrep.data(), sizeof(int32_t) * K, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && b->d_need)
    e = cudaMemcpy(b->d_need, lneed.data(), sizeof(uint32_t) * K, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(b->d_pats);
    cudaFree(b->d_mp);
    cudaFree(b->d_rep);
    cudaFree(b->d_need);
    delete b;
    return e == cudaErrorMemoryAllocation ? fail(MB_ENOMEM, "batch upload alloc") : cuda_fail(e, "batch upload");
  }
  *out = b;
  return MB_OK;
}

void mb_batch_destroy(mb_batch* b) {
  if (!b) return;
  cudaFree(b->d_pats);
  cudaFree(b->d_mp);
  cudaFree(b->d_rep);
  cudaFree(b->d_need);
  delete b;
}

int mb_find_batch_prepared(mb_ctx* c, const mb_batch* b, const uint8_t* d_text, int64_t n, int64_t* d_out,
                           int64_t cap, int64_t* d_offsets, void* stream) {
  if (!c || !b || !d_offsets) return fail(MB_EINVAL, "bad argument");
  if (n < 0 || cap < 0) return fail(MB_EINVAL, "negative size");
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev != b->device) return fail(MB_EINVAL, "batch was prepared on another device");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ctx_enter(c, st);
  if (rc) return rc;
  if ((rc = stage_begin(c))) return rc;
  rc = run_batch(c, b->d_pats, b->h_pats.data(), b->K, d_text, n, d_out, cap, d_offsets, st, &b->pass, b->d_mp,
                 b->src.data(), b->d_rep, b->d_need);
  if (rc) tickets_recover(c, st);
  const int rc2 = stage_end(c, st);
  const int rc3 = ctx_leave(c, st);
  return rc ? rc : rc2 ? rc2 : rc3;
}

int mb_histogram(mb_ctx* c, const uint8_t* d_text, int64_t n, int64_t* d_hist, void* stream) {
  if (!c || !d_hist) return fail(MB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = -1;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev != c->device) return fail(MB_EINVAL, "current CUDA device differs from the context's device");
  CUDA_TRY(cudaMemsetAsync(d_hist, 0, 256 * sizeof(int64_t), st));
  if (n <= 0) return MB_OK;
  // per-warp counters are 32-bit: a warp sees at most n / (warps in the grid) + 64 KiB bytes
  int64_t blocks = std::min<int64_t>((n + 65535) / 65536, (int64_t)c->nsm * 8);
  blocks = std::max<int64_t>(blocks, (n >> 31) + 1);
  hist_kernel<<<(int)blocks, HIST_WARPS * 32, 0, st>>>(d_text, n, (unsigned long long*)d_hist);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

static int ensure_host_bufs(mb_ctx* c, int64_t n, int64_t outcap, int64_t nofs) {
  if (!c->stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  if (n > c->text_cap) {
    cudaFree(c->d_text);
    c->d_text = nullptr;
    if (cudaMalloc(&c->d_text, n + 16) != cudaSuccess) {
      c->text_cap = 0;
      return fail(MB_ENOMEM, "text buffer alloc");
    }
    c->text_cap = n;
  }
  if (outcap > c->out_cap) {
    cudaFree(c->d_out);
    c->d_out = nullptr;
    if (cudaMalloc(&c->d_out, sizeof(int64_t) * outcap) != cudaSuccess) {
      c->out_cap = 0;
      return fail(MB_ENOMEM, "output buffer alloc");
    }
    c->out_cap = outcap;
  }
  if (nofs > c->offs_cap) {
    cudaFree(c->d_offs);
    c->d_offs = nullptr;
    if (cudaMalloc(&c->d_offs, sizeof(int64_t) * nofs) != cudaSuccess) {
      c->offs_cap = 0;
      return fail(MB_ENOMEM, "offsets alloc");
    }
    c->offs_cap = nofs;
  }
  return MB_OK;
}

int mb_search_batch_host(mb_ctx* c, const uint8_t* const* h_patterns, const int64_t* ms, int K,
                         const uint8_t* h_text, int64_t n, int64_t* h_out, int64_t cap, int64_t* h_offsets) {
  if (!c || !h_patterns || !ms || K < 1 || !h_offsets) return fail(MB_EINVAL, "bad argument");
  // host buffers in and out: run on the context's device whatever is current
  DeviceGuard guard(c->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  if (n < 0 || cap < 0 || (n > 0 && !h_text)) return fail(MB_EINVAL, "bad text");
  // plans come from the context's cache (created and uploaded on first use;
  // the cache is dropped wholesale past 4096 patterns)
  std::vector<mb_plan*> plans(K, nullptr);
  if (c->host_plans.size() + (size_t)K > 4096) {
    for (auto& kv : c->host_plans) mb_plan_destroy(kv.second);
    c->host_plans.clear();
  }
  for (int k = 0; k < K; k++) {
    if (ms[k] < 0 || (ms[k] > 0 && !h_patterns[k])) return fail(MB_EINVAL, "bad pattern");
    std::string key(reinterpret_cast<const char*>(h_patterns[k]), (size_t)ms[k]);
    auto it = c->host_plans.find(key);
    if (it != c->host_plans.end()) {
      plans[k] = it->second;
      continue;
    }
    int rc = mb_plan_create(h_patterns[k], ms[k], nullptr, &plans[k]);
    if (rc) return rc;
    c->host_plans.emplace(std::move(key), plans[k]);
  }
  int rc = ensure_host_bufs(c, n, std::max<int64_t>(cap, 1), K + 1);
  if (rc) return rc;
  cudaStream_t st = c->stream;
  if (n > 0) CUDA_TRY(cudaMemcpyAsync(c->d_text, h_text, n, cudaMemcpyHostToDevice, st));
  rc = mb_find_batch(c, plans.data(), K, c->d_text, n, c->d_out, cap, c->d_offs, st);
  if (rc) {
    cudaStreamSynchronize(st);  // the upload may still read h_text
    return rc;
  }
  // the first EAGER positions come back with the offsets, before the one
  // synchronisation (entries past the count are don't-care); the rest, if
  // any, once the count is known
  const int64_t eager = std::min<int64_t>(cap, (int64_t)1 << 16);
  cudaError_t e = cudaMemcpyAsync(h_offsets, c->d_offs, sizeof(int64_t) * (K + 1), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && eager > 0)
    e = cudaMemcpyAsync(h_out, c->d_out, sizeof(int64_t) * eager, cudaMemcpyDeviceToHost, st);
  const cudaError_t es = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "result copy");
  if (es != cudaSuccess) return cuda_fail(es, "batch search");
  const int64_t total = h_offsets[K];
  const int64_t ncopy = std::min(total, cap);
  if (ncopy > eager) {
    e = cudaMemcpy(h_out + eager, c->d_out + eager, sizeof(int64_t) * (ncopy - eager), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "position copy");
  }
  if (total > cap) return fail(MB_EOVERFLOW, "output capacity too small");
  return MB_OK;
}

int mb_search_host(mb_ctx* c, const uint8_t* h_pattern, int64_t m, const uint8_t* h_text, int64_t n,
                   int64_t* h_out, int64_t cap, int64_t* h_count) {
  if (!h_count) return fail(MB_EINVAL, "null count");
  int64_t offs[2] = {0, 0};
  int rc = mb_search_batch_host(c, &h_pattern, &m, 1, h_text, n, h_out, cap, offs);
  *h_count = offs[1];
  return rc;
}

}  // extern "C"

// Trace build only (make trace): copy out the kernel-phase timestamps
// (device_common.cuh MB_TRACE_MARK) and optionally re-arm them.
extern "C" int mb_debug_trace(uint64_t* out, int reset) {
#ifdef MB_TRACE
  if (out) CUDA_TRY(cudaMemcpyFromSymbol(out, g_trace, sizeof(uint64_t) * 32));
  if (reset) {
    uint64_t init[32];
    for (int i = 0; i < 32; i++) init[i] = (i & 1) ? 0ULL : ~0ULL;
    CUDA_TRY(cudaMemcpyToSymbol(g_trace, init, sizeof(init)));
  }
  return MB_OK;
#else
  (void)out, (void)reset;
  return fail(MB_EINVAL, "not a trace build");
#endif
}
