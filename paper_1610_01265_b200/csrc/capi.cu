// C ABI of libsts_b200 (include/sts_b200.h): grid handle + metrics, halo
// exchange (virtual slabs / NCCL), and the host drivers of the RKL2 and
// BE+Jacobi-PCG advances.  Every arithmetic step of the path runs in the
// kernels of stencil.cu / aux.cu; the host only sequences launches, computes
// the per-stage RKL2 scalars, and polls PCG convergence flags.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

#include "sts_common.cuh"

namespace sts {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

template <class F>
static int guard(F&& f) {
  try {
    f();
    return STS_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return STS_ERR_ALLOC;
  } catch (const std::exception& e) {
    set_error(e.what());
    return STS_ERR_STATE;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    STS_CUDA(cudaGetDevice(&prev));
    if (prev != dev) STS_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

Geo slab_geo(const sts_grid* g, const Slab& s) {
  Geo G;
  G.n1g = g->n1g;
  G.n2 = g->n2;
  G.n3 = g->n3;
  G.periodic3 = g->periodic3;
  G.i0 = s.i0;
  G.nl = s.nl;
  G.plane = g->plane;
  G.cstride = (long long)g->nl * g->plane;
  G.m = g->m;
  return G;
}

static cudaEvent_t get_event(sts_grid* g) {
  if (!g->free_events.empty()) {
    cudaEvent_t e = g->free_events.back();
    g->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  STS_CUDA(cudaEventCreate(&e));
  return e;
}

// brackets one launch (or exchange) with events when timing is enabled; counts launches
struct Timed {
  sts_grid* g;
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  bool count;
  Timed(sts_grid* g_, int kind_, cudaStream_t st_, bool count_ = true) : g(g_), kind(kind_), st(st_), count(count_) {
    if (g->timing) {
      a = get_event(g);
      STS_CUDA(cudaEventRecord(a, st));
    }
  }
  ~Timed() {
    if (a) {
      cudaEvent_t b = get_event(g);
      cudaEventRecord(b, st);
      g->pending.push_back({kind, a, b});
    }
    if (count) g->launches += 1;
  }
};

static int stencil_kind(int mode, int epi) { return (mode == STS_MODE_ANISO ? STS_K_ANISO_F : STS_K_ISO_F) + epi; }

static void collect_timing(sts_grid* g) {
  for (auto& r : g->pending) {
    STS_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    STS_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    g->acc_ms[r.kind] += ms;
    g->acc_n[r.kind] += 1;
    g->free_events.push_back(r.a);
    g->free_events.push_back(r.b);
  }
  g->pending.clear();
}

double* ws_get(sts_grid* g, size_t bytes) {
  if (bytes <= g->ws.bytes) return g->ws.base;
  if (g->ws.base) STS_CUDA(cudaFree(g->ws.base));
  g->ws.base = nullptr;
  g->ws.bytes = 0;
  if (cudaMalloc(&g->ws.base, bytes) != cudaSuccess) {
    cudaGetLastError();
    throw Error{STS_ERR_ALLOC, "cudaMalloc of " + std::to_string(bytes) + " bytes of workspace failed"};
  }
  g->ws.bytes = bytes;
  return g->ws.base;
}

static void ensure_red(sts_grid* g, size_t bytes) {
  if (bytes <= g->red_bytes) return;
  if (g->d_red) STS_CUDA(cudaFree(g->d_red));
  g->d_red = nullptr;
  g->red_bytes = 0;
  if (cudaMalloc(&g->d_red, bytes) != cudaSuccess) {
    cudaGetLastError();
    throw Error{STS_ERR_ALLOC, "cudaMalloc of reduction buffer failed"};
  }
  g->red_bytes = bytes;
}

// ----------------------------------------------------------------------------
// halo buffers and exchange
// ----------------------------------------------------------------------------
static void ensure_halos(sts_grid* g) {
  for (auto& s : g->slabs) {
    if (!s.halo_lo.empty()) continue;
    s.halo_lo.assign(H_NSLOTS, nullptr);
    s.halo_hi.assign(H_NSLOTS, nullptr);
    if (!s.has_lo && !s.has_hi) continue;
    const size_t side = (size_t)MAXC * g->plane;
    for (int h = 0; h < H_NSLOTS; ++h) {
      double* base = nullptr;
      STS_CUDA(cudaMalloc(&base, 2 * side * sizeof(double)));
      STS_CUDA(cudaMemset(base, 0, 2 * side * sizeof(double)));
      g->halo_bytes += 2 * side * sizeof(double);
      s.halo_lo[h] = base;          // freed through halo_lo
      s.halo_hi[h] = base + side;
    }
  }
}

static bool needs_halos(const sts_grid* g) {
  for (auto& s : g->slabs)
    if (s.has_lo || s.has_hi) return true;
  return false;
}

// Fill the `slot` halo planes of every slab from `arr` ([ncomp][nl][plane], device).
//  * slabs of this process (virtual decomposition): device-to-device copies
//  * neighbouring ranks: ncclSend / ncclRecv of one plane per component
static void exchange(sts_grid* g, int slot, const double* arr, int ncomp, cudaStream_t st) {
  if (!needs_halos(g)) return;
  if (g->comm == nullptr && g->n_virtual == 1)
    throw Error{STS_ERR_STATE, "this handle is an r-slab of a distributed grid (i0 > 0 or i0 + nl < n1): "
                               "call sts_comm_init before any operator"};
  ensure_halos(g);
  Timed t(g, STS_K_HALO, st, false);
  const long long P = g->plane;
  const long long cs = (long long)g->nl * P;
  if (g->comm == nullptr) {
    for (auto& s : g->slabs) {
      if (s.has_lo)
        STS_CUDA(cudaMemcpy2DAsync(s.halo_lo[slot], P * sizeof(double), arr + s.off - P, cs * sizeof(double),
                                   P * sizeof(double), ncomp, cudaMemcpyDeviceToDevice, st));
      if (s.has_hi)
        STS_CUDA(cudaMemcpy2DAsync(s.halo_hi[slot], P * sizeof(double), arr + s.off + (long long)s.nl * P,
                                   cs * sizeof(double), P * sizeof(double), ncomp, cudaMemcpyDeviceToDevice, st));
    }
    return;
  }
  Slab& s = g->slabs[0];
  STS_NCCL(ncclGroupStart());
  for (int c = 0; c < ncomp; ++c) {
    if (s.has_lo) {
      STS_NCCL(ncclRecv(s.halo_lo[slot] + c * P, P, ncclDouble, g->rank - 1, g->comm, st));
      STS_NCCL(ncclSend(arr + c * cs, P, ncclDouble, g->rank - 1, g->comm, st));
    }
    if (s.has_hi) {
      STS_NCCL(ncclRecv(s.halo_hi[slot] + c * P, P, ncclDouble, g->rank + 1, g->comm, st));
      STS_NCCL(ncclSend(arr + c * cs + (long long)(s.nl - 1) * P, P, ncclDouble, g->rank + 1, g->comm, st));
    }
  }
  STS_NCCL(ncclGroupEnd());
}

static FieldV view(const sts_grid* g, const Slab& s, int slot, const double* arr) {
  FieldV f;
  f.p = arr ? arr + s.off : nullptr;
  f.lo = (arr && s.has_lo) ? s.halo_lo[slot] : nullptr;
  f.hi = (arr && s.has_hi) ? s.halo_hi[slot] : nullptr;
  return f;
}

// ----------------------------------------------------------------------------
// host-array path (include/sts_b200.h "Array arguments"): every host array is staged
// through a device buffer of the handle's staging pool.  Uploads run on the handle's
// H2D copy stream and downloads on its D2H copy stream, so a call's copies overlap the
// compute of the calls enqueued before / after it; the compute stream waits only for
// its own inputs.  Pinned host arrays make the call asynchronous (like cudaMemcpyAsync:
// the caller keeps inputs unchanged and reads outputs after sts_grid_join /
// sts_grid_synchronize); a pageable array makes it synchronous.
// ----------------------------------------------------------------------------
enum class Mem { Device, Pinned, Pageable };

static Mem mem_kind(const void* p) {
  if (!p) return Mem::Device;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return Mem::Pageable;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return Mem::Device;
  return a.type == cudaMemoryTypeHost ? Mem::Pinned : Mem::Pageable;
}

static bool is_device_ptr(const void* p) { return mem_kind(p) == Mem::Device; }

static cudaStream_t copy_stream(sts_grid* g, bool h2d) {
  cudaStream_t& s = h2d ? g->h2d_stream : g->d2h_stream;
  cudaEvent_t& e = h2d ? g->ev_h2d_last : g->ev_d2h_last;
  if (!s) STS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  if (!e) STS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return s;
}

static void pool_reclaim(sts_grid* g) {
  for (auto& b : g->stage_pool) {
    if (!b.pending || b.claimed) continue;
    const cudaError_t q = cudaEventQuery(b.ev);
    if (q == cudaSuccess) b.pending = false;
    else if (q != cudaErrorNotReady) STS_CUDA(q);
  }
}

static void pool_free_idle(sts_grid* g) {
  for (auto it = g->stage_pool.begin(); it != g->stage_pool.end();) {
    if (!it->pending && !it->claimed) {
      cudaFree(it->p);
      cudaEventDestroy(it->ev);
      g->stage_bytes -= it->bytes;
      it = g->stage_pool.erase(it);
    } else {
      ++it;
    }
  }
}

// (a staging allocation leaves STAGE_HEADROOM bytes of the device free for everything else)
constexpr size_t STAGE_HEADROOM = 6ull << 30;
static double* try_alloc(size_t bytes, bool headroom = true) {
  double* p = nullptr;
  size_t fr = 0, tot = 0;
  if (headroom && cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr < bytes + STAGE_HEADROOM) return nullptr;
  if (cudaMalloc(&p, bytes) == cudaSuccess) return p;
  cudaGetLastError();
  return nullptr;
}

// a staging buffer of >= bytes that no enqueued work still uses: a free one; else a new
// one; else (device full) the OLDEST in-flight one large enough, waited for -- which
// bounds the pool without a device-wide synchronization; only when no buffer is large
// enough are all of them waited for and the idle ones released (cudaFree synchronizes)
static StageBuf* stage_acquire(sts_grid* g, size_t bytes) {
  bytes = (bytes + 255) / 256 * 256;
  pool_reclaim(g);
  StageBuf* best = nullptr;
  for (auto& b : g->stage_pool)
    if (!b.pending && !b.claimed && b.bytes >= bytes && (!best || b.bytes < best->bytes)) best = &b;
  if (!best) {
    if (double* p = try_alloc(bytes)) {
      StageBuf nb;
      nb.p = p;
      nb.bytes = bytes;
      STS_CUDA(cudaEventCreateWithFlags(&nb.ev, cudaEventDisableTiming));
      g->stage_pool.push_back(nb);
      g->stage_bytes += bytes;
      best = &g->stage_pool.back();
    }
  }
  if (!best) {
    StageBuf* old = nullptr;
    for (auto& b : g->stage_pool)
      if (b.pending && !b.claimed && b.bytes >= bytes && (!old || b.seq < old->seq)) old = &b;
    if (old) {
      STS_CUDA(cudaEventSynchronize(old->ev));
      old->pending = false;
      best = old;
    }
  }
  if (!best) {
    for (auto& b : g->stage_pool)
      if (b.pending && !b.claimed) STS_CUDA(cudaEventSynchronize(b.ev));
    pool_reclaim(g);
    pool_free_idle(g);
    if (double* p = try_alloc(bytes, false)) {
      StageBuf nb;
      nb.p = p;
      nb.bytes = bytes;
      STS_CUDA(cudaEventCreateWithFlags(&nb.ev, cudaEventDisableTiming));
      g->stage_pool.push_back(nb);
      g->stage_bytes += bytes;
      best = &g->stage_pool.back();
    }
  }
  if (!best) throw Error{STS_ERR_ALLOC, "cudaMalloc of " + std::to_string(bytes) + " bytes of host-array staging failed"};
  best->claimed = true;
  return best;
}

// mapped-mailbox word of the Gershgorin maximum (the PCG scalars use the words before it)
constexpr int DT_MAILBOX = 64;

struct HostIO {
  sts_grid* g;
  cudaStream_t st;
  struct Arr {
    const double* host;
    double** slot;    // the call's pointer variable, rewritten to the staging buffer
    size_t n;
    StageBuf* buf;
  };
  std::vector<Arr> ins, outs;
  bool sync = false;  // a pageable array: the call returns with its outputs written back
  bool ended = false;

  HostIO(sts_grid* g_, cudaStream_t st_) : g(g_), st(st_) {}
  void input(const double*& p, size_t n) {
    const Mem k = mem_kind(p);
    if (k == Mem::Device) return;
    sync = sync || k == Mem::Pageable;
    ins.push_back({p, const_cast<double**>(&p), n, nullptr});
  }
  void output(double*& p, size_t n) {
    const Mem k = mem_kind(p);
    if (k == Mem::Device) return;
    sync = sync || k == Mem::Pageable;
    outs.push_back({p, &p, n, nullptr});
  }
  bool any() const { return !ins.empty() || !outs.empty(); }
  // claim staging buffers, start the uploads, make the compute stream wait for them
  void begin() {
    if (!ins.empty()) {
      cudaStream_t cs = copy_stream(g, true);
      for (auto& a : ins) {
        a.buf = stage_acquire(g, a.n * sizeof(double));
        STS_CUDA(cudaMemcpyAsync(a.buf->p, a.host, a.n * sizeof(double), cudaMemcpyHostToDevice, cs));
        *a.slot = a.buf->p;
      }
      STS_CUDA(cudaEventRecord(g->ev_h2d_last, cs));
      STS_CUDA(cudaStreamWaitEvent(st, g->ev_h2d_last, 0));
      g->h2d_used = true;
    }
    for (auto& a : outs) {
      a.buf = stage_acquire(g, a.n * sizeof(double));
      *a.slot = a.buf->p;
    }
  }
  // after the call's kernels: release the inputs (free once the kernels ran), download
  // the outputs on the D2H stream (free once downloaded)
  void end() {
    ended = true;
    for (auto& a : ins) release(a.buf, st);
    if (!outs.empty()) {
      cudaStream_t cs = copy_stream(g, false);
      StageBuf* first = outs[0].buf;
      STS_CUDA(cudaEventRecord(first->ev, st));   // (reused below as the D2H buffer's own event)
      STS_CUDA(cudaStreamWaitEvent(cs, first->ev, 0));
      for (auto& a : outs) {
        STS_CUDA(cudaMemcpyAsync(const_cast<double*>(a.host), a.buf->p, a.n * sizeof(double), cudaMemcpyDeviceToHost,
                                 cs));
        release(a.buf, cs);
      }
      STS_CUDA(cudaEventRecord(g->ev_d2h_last, cs));
      g->d2h_used = true;
      if (sync) STS_CUDA(cudaStreamSynchronize(cs));
    }
    if (sync) STS_CUDA(cudaStreamSynchronize(st));
  }
  void release(StageBuf* b, cudaStream_t s) {
    if (!b) return;
    STS_CUDA(cudaEventRecord(b->ev, s));
    b->pending = true;
    b->claimed = false;
    b->seq = ++g->stage_seq;
  }
  ~HostIO() {
    if (ended) return;   // an error path: whatever was enqueued may still read the buffers
    for (auto* v : {&ins, &outs})
      for (auto& a : *v)
        if (a.buf) {
          if (cudaEventRecord(a.buf->ev, st) == cudaSuccess) a.buf->pending = true;
          a.buf->claimed = false;
        }
    cudaGetLastError();
  }
};

static void check_mode(int mode, int ncomp, const double* b) {
  STS_REQUIRE(mode == STS_MODE_ISO || mode == STS_MODE_ANISO, "mode must be STS_MODE_ISO or STS_MODE_ANISO");
  STS_REQUIRE(ncomp >= 1 && ncomp <= MAXC, "ncomp must be 1..3");
  STS_REQUIRE(mode == STS_MODE_ISO || ncomp == 1, "STS_MODE_ANISO supports ncomp == 1");
  STS_REQUIRE(mode == STS_MODE_ISO || b != nullptr, "STS_MODE_ANISO requires b");
}

// ----------------------------------------------------------------------------
// resident coefficients (sts_grid_bind_coeffs): one slot per operator mode
// ----------------------------------------------------------------------------
static int slot_index(int mode) { return mode == STS_MODE_ANISO ? 1 : 0; }

// the bound arrays changed: the derived data must be rebuilt
static void slot_invalidate(CoefSlot& s) {
  s.ev_ok = s.pre_ok = false;
  s.lam = -1.0;
}

static void slot_free(CoefSlot& s) {
  for (int i = 0; i < 5; ++i) {
    if (s.own[i]) cudaFree(s.own[i]);
    s.own[i] = nullptr;
    s.own_n[i] = 0;
  }
  for (int d = 0; d < 3; ++d) {
    if (s.kfk[d]) cudaFree(s.kfk[d]);
    s.kfk[d] = nullptr;
  }
  if (s.dbuf) cudaFree(s.dbuf);
  s.dbuf = nullptr;
  s.dbytes = 0;
  if (s.last_use) cudaEventDestroy(s.last_use);
  s.last_use = nullptr;
  s.use_set = false;
  s.user_dev = false;
  s.k[0] = s.k[1] = s.k[2] = s.b = s.w = nullptr;
  s.bound = false;
  slot_invalidate(s);
}

static double* dev_alloc(size_t n, const char* what) {
  double* p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    throw Error{STS_ERR_ALLOC, std::string("cudaMalloc of ") + what + " failed"};
  }
  return p;
}

// the binding's derived-data buffer, at least n doubles
static double* slot_dbuf(CoefSlot& s, size_t n) {
  if (s.dbytes < n * sizeof(double)) {
    if (s.dbuf) STS_CUDA(cudaFree(s.dbuf));
    s.dbuf = nullptr;
    s.dbuf = dev_alloc(n, "resident derived coefficients");
    s.dbytes = n * sizeof(double);
  }
  return s.dbuf;
}

// `ws`, a stream about to overwrite the binding's arrays, waits for their last readers
static void slot_wait_readers(CoefSlot& s, cudaStream_t ws) {
  if (s.use_set) STS_CUDA(cudaStreamWaitEvent(ws, s.last_use, 0));
}

// a call on stream `st` has enqueued its reads of the binding
static void slot_used(CoefSlot* s, cudaStream_t st) {
  if (!s) return;
  if (!s->last_use) STS_CUDA(cudaEventCreateWithFlags(&s->last_use, cudaEventDisableTiming));
  STS_CUDA(cudaEventRecord(s->last_use, st));
  s->use_set = true;
}

// a bound array the caller owns (written on the caller's stream, not by the library)
static bool slot_user_array(const CoefSlot& s, const double* p) {
  if (!p) return false;
  for (int i = 0; i < 5; ++i)
    if (p == s.own[i]) return false;
  for (int d = 0; d < 3; ++d)
    if (p == s.kfk[d]) return false;
  return true;
}

static void slot_update_user_dev(CoefSlot& s) {
  s.user_dev = slot_user_array(s, s.k[0]) || slot_user_array(s, s.k[1]) || slot_user_array(s, s.k[2]) ||
               slot_user_array(s, s.b) || slot_user_array(s, s.w);
}

static cudaStream_t coef_stream(sts_grid* g) {
  if (!g->coef_stream) STS_CUDA(cudaStreamCreateWithFlags(&g->coef_stream, cudaStreamNonBlocking));
  if (!g->ev_coef) STS_CUDA(cudaEventCreateWithFlags(&g->ev_coef, cudaEventDisableTiming));
  if (!g->ev_pos) STS_CUDA(cudaEventCreateWithFlags(&g->ev_pos, cudaEventDisableTiming));
  return g->coef_stream;
}

// The coefficient arrays one call uses (device pointers): the caller's arrays (staged
// if on the host), or the mode's resident binding when k1 = k2 = k3 = NULL.
struct Coefs {
  const double *k1 = nullptr, *k2 = nullptr, *k3 = nullptr, *b = nullptr, *w = nullptr;
  CoefSlot* slot = nullptr;
};

// (io keeps pointers to c's fields: c must outlive io.begin())
static void resolve_coefs(Coefs& c, sts_grid* g, int mode, const double* k1, const double* k2, const double* k3,
                          const double* b, const double* w, HostIO& io, size_t N) {
  if (!k1 && !k2 && !k3) {
    CoefSlot& s = g->slot[slot_index(mode)];
    STS_REQUIRE(s.bound && s.k[0] && s.k[1] && s.k[2],
                "k1 = k2 = k3 = NULL selects the resident coefficients, but none are bound for this mode "
                "(sts_grid_bind_coeffs / sts_face_kappa_spitzer with NULL outputs)");
    STS_REQUIRE(!b && !w, "with resident coefficients (k = NULL) b and w must be NULL too (they are bound)");
    STS_REQUIRE(mode == STS_MODE_ISO || s.b, "the resident STS_MODE_ANISO coefficients have no b bound");
    c.k1 = s.k[0];
    c.k2 = s.k[1];
    c.k3 = s.k[2];
    c.b = mode == STS_MODE_ANISO ? s.b : nullptr;
    c.w = s.w;
    c.slot = &s;
    return;
  }
  STS_REQUIRE(k1 && k2 && k3, "k1, k2, k3 must all be given (or all NULL for the resident coefficients)");
  c.k1 = k1;
  c.k2 = k2;
  c.k3 = k3;
  c.b = mode == STS_MODE_ANISO ? b : nullptr;
  c.w = w;
  io.input(c.k1, N);
  io.input(c.k2, N);
  io.input(c.k3, N);
  if (mode == STS_MODE_ANISO) io.input(c.b, 3 * N);
  io.input(c.w, N);
}

// coefficient halos for the operator (once per call)
static void exchange_coeffs(sts_grid* g, int mode, const double* k1, const double* k2, const double* k3,
                            const double* b, cudaStream_t st) {
  exchange(g, H_K1, k1, 1, st);
  if (mode == STS_MODE_ANISO) {
    exchange(g, H_K2, k2, 1, st);
    exchange(g, H_K3, k3, 1, st);
    exchange(g, H_B, b, 3, st);
  }
}

static StencilCall make_call(sts_grid* g, const Slab& s, int mode, int ncomp, int epi, const double* u,
                             const double* k1, const double* k2, const double* k3, const double* b,
                             const double* w) {
  StencilCall c{};
  c.mode = mode;
  c.ncomp = ncomp;
  c.epi = epi;
  c.geo = slab_geo(g, s);
  c.u = view(g, s, H_U, u);
  c.k1 = view(g, s, H_K1, k1);
  c.k2 = view(g, s, H_K2, k2);
  c.k3 = view(g, s, H_K3, k3);
  c.b = view(g, s, H_B, b);
  c.w = w ? w + s.off : nullptr;
  c.ib = 0;
  c.ie = s.nl;
  return c;
}

// workspace carving unit: every scratch field starts on a 256 B boundary (TMA needs 16 B)
static size_t rnd(size_t n) { return (n + 31) / 32 * 32; }

static size_t vertex_coef_doubles(const sts_grid* g, int mode) {
  if (mode != STS_MODE_ANISO) return 0;
  size_t n = 0;
  for (auto& s : g->slabs) n += rnd(3 * (size_t)ev_cstride(s.nl, g->n2, g->n3));
  return n;
}

// per-advance precompute of the frozen vertex coefficients (after exchange_coeffs)
static std::vector<const double*> build_vertex_coefs(sts_grid* g, int mode, double* base, const double* k1,
                                                     const double* k2, const double* k3, const double* b,
                                                     cudaStream_t st) {
  std::vector<const double*> out(g->slabs.size(), nullptr);
  if (mode != STS_MODE_ANISO) return out;
  size_t o = 0;
  for (size_t i = 0; i < g->slabs.size(); ++i) {
    const Slab& s = g->slabs[i];
    out[i] = base + o;
    Timed t(g, STS_K_VERTEX_COEF, st);
    launch_vertex_coef(slab_geo(g, s), view(g, s, H_B, b), view(g, s, H_K1, k1), view(g, s, H_K2, k2),
                       view(g, s, H_K3, k3), base + o, st);
    o += rnd(3 * (size_t)ev_cstride(s.nl, g->n2, g->n3));
  }
  return out;
}

// one stencil pass: the TMA pipelined kernel where eligible, else the cp.async kernels
static void launch_pass(sts_grid* g, const StencilCall& c, cudaStream_t st) {
  const bool aniso = c.mode == STS_MODE_ANISO;
  const int kind = (c.epi == EPI_PCG_S)         ? (aniso ? STS_K_ANISO_PCG_S : STS_K_ISO_PCG_S)
                   : (c.epi == EPI_PCG_M)       ? (aniso ? STS_K_ANISO_PCG_M : STS_K_ISO_PCG_M)
                   : (c.epi == EPI_RKL2_DSTAGE) ? (aniso ? STS_K_ANISO_RKL2_DSTAGE : STS_K_ISO_RKL2_DSTAGE)
                                                : stencil_kind(c.mode, c.epi);
  Timed t(g, kind, st);
  if (g->tma && (launch_aniso_tma(c, st) || launch_iso_tma(c, st))) return;
  if (c.epi == EPI_PCG_S || c.epi == EPI_PCG_M || c.epi == EPI_RKL2_DSTAGE)
    throw Error{STS_ERR_STATE, "TMA-only pass launched without a TMA-eligible call"};
  launch_stencil(c, st);
}

static double* off(double* p, const Slab& s) { return p ? p + s.off : nullptr; }

// CTAs one pass over local planes [c.ib, c.ie) launches (sizes the partial-sum rows)
static int pass_blocks(const sts_grid* g, const StencilCall& c) {
  if (g->tma && aniso_tma_eligible(c)) return aniso_tma_blocks(c);
  if (g->tma && iso_tma_eligible(c)) return iso_tma_blocks(c);
  return stencil_blocks(c.mode, c.epi, c.geo, c.ib, c.ie);
}

static cudaStream_t comm_stream(sts_grid* g) {
  if (!g->comm_stream) {
    int lo = 0, hi = 0;
    STS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    STS_CUDA(cudaStreamCreateWithPriority(&g->comm_stream, cudaStreamNonBlocking, hi));
  }
  if (!g->ev_a) STS_CUDA(cudaEventCreateWithFlags(&g->ev_a, cudaEventDisableTiming));
  if (!g->ev_b) STS_CUDA(cudaEventCreateWithFlags(&g->ev_b, cudaEventDisableTiming));
  return g->comm_stream;
}

// the library's own non-blocking stream for CUDA-graph capture / replay
static cudaStream_t graph_stream(sts_grid* g) {
  if (!g->graph_stream) STS_CUDA(cudaStreamCreateWithFlags(&g->graph_stream, cudaStreamNonBlocking));
  if (!g->ev_c) STS_CUDA(cudaEventCreateWithFlags(&g->ev_c, cudaEventDisableTiming));
  return g->graph_stream;
}

struct Xch {
  int slot;
  const double* arr;
  int ncomp;
};

// plane ranges of one sweep, in launch order: every slab's interior planes (which
// read no halo) first, then the boundary planes next to a neighbour slab
struct Range {
  size_t si;
  int ib, ie;
  bool boundary;
};
static std::vector<Range> sweep_ranges(const sts_grid* g, bool overlap) {
  std::vector<Range> v;
  for (size_t si = 0; si < g->slabs.size(); ++si) {
    const Slab& s = g->slabs[si];
    if (!overlap) {
      v.push_back({si, 0, s.nl, false});
      continue;
    }
    const int lo = s.has_lo ? 1 : 0, hi = s.has_hi ? s.nl - 1 : s.nl;
    if (hi > lo) v.push_back({si, lo, hi, false});
  }
  if (overlap)
    for (size_t si = 0; si < g->slabs.size(); ++si) {
      const Slab& s = g->slabs[si];
      const int lo = s.has_lo ? 1 : 0;
      if (s.has_lo) v.push_back({si, 0, std::min(1, s.nl), true});
      if (s.has_hi && s.nl - 1 >= lo) v.push_back({si, s.nl - 1, s.nl, true});
    }
  return v;
}

// One stencil pass over every slab whose source fields `xs` need halo planes
// (DESIGN.md §6): the halo exchange runs on the high-priority communication
// stream (NCCL send/recv between ranks, device copies between virtual slabs)
// while the interior planes are computed on `st`; the boundary planes follow once
// the halos have landed.  `make(si)` returns the slab's StencilCall; returns the
// number of CTAs launched (per-CTA partial sums are written from pbase 0 on).
template <class Make>
static int sweep(sts_grid* g, std::initializer_list<Xch> xs, cudaStream_t st, Make make,
                 const FinRed* fin = nullptr) {
  // halo exchange on the communication stream; with halo_overlap the interior planes are
  // computed meanwhile and the boundary planes after it (one-plane launches), else the
  // exchange is waited for and each slab is ONE launch (the one-plane
  // launches cost more than the exchange they hide)
  const bool exch = needs_halos(g) && xs.size() > 0;
  const bool overlap = exch && g->halo_overlap;
  cudaStream_t cst = nullptr;
  if (exch) {
    g->comm_local += 1;
    cst = comm_stream(g);
    STS_CUDA(cudaEventRecord(g->ev_a, st));
    STS_CUDA(cudaStreamWaitEvent(cst, g->ev_a, 0));
    for (const Xch& x : xs) exchange(g, x.slot, x.arr, x.ncomp, cst);
    STS_CUDA(cudaEventRecord(g->ev_b, cst));
    if (!overlap) STS_CUDA(cudaStreamWaitEvent(st, g->ev_b, 0));
  }
  const std::vector<Range> ranges = sweep_ranges(g, overlap);
  std::vector<StencilCall> calls;
  int total = 0;
  for (const Range& r : ranges) {
    StencilCall c = make(r.si);
    c.ib = r.ib;
    c.ie = r.ie;
    c.ea.pbase = total;
    total += pass_blocks(g, c);
    calls.push_back(c);
  }
  bool waited = false;
  for (size_t i = 0; i < calls.size(); ++i) {
    if (ranges[i].boundary && !waited) {
      STS_CUDA(cudaStreamWaitEvent(st, g->ev_b, 0));
      waited = true;
    }
    if (fin && i + 1 == calls.size()) {   // the last launch finishes the pass's reduction
      calls[i].ea.fin = *fin;
      calls[i].ea.fin.ntot = total;
    }
    launch_pass(g, calls[i], st);
  }
  if (overlap && !waited) STS_CUDA(cudaStreamWaitEvent(st, g->ev_b, 0));
  return total;
}

// CTAs of a sweep (same ranges and kernel choice as sweep())
template <class Make>
static int sweep_blocks(sts_grid* g, bool has_x, Make make) {
  int pb = 0;
  for (const Range& r : sweep_ranges(g, needs_halos(g) && has_x && g->halo_overlap)) {
    StencilCall c = make(r.si);
    c.ib = r.ib;
    c.ie = r.ie;
    pb += pass_blocks(g, c);
  }
  return pb;
}


static const double* off(const double* p, const Slab& s) { return p ? p + s.off : nullptr; }

// RKL2 coefficients, PAPER.md:134-138 (gamma~ per DESIGN R6)
struct Rkl2Coef {
  std::vector<double> mu, nu, mut, gt;
};
static Rkl2Coef rkl2_coefs(int s) {
  std::vector<double> bj(s + 1);
  for (int j = 0; j <= s; ++j) bj[j] = (j <= 2) ? 1.0 / 3.0 : (double(j) * j + j - 2.0) / (2.0 * j * (j + 1.0));
  Rkl2Coef c;
  c.mu.assign(s + 1, 0.0);
  c.nu.assign(s + 1, 0.0);
  c.mut.assign(s + 1, 0.0);
  c.gt.assign(s + 1, 0.0);
  const double ss = double(s) * s + s - 2.0;
  c.mut[1] = 4.0 / (3.0 * ss);
  for (int j = 2; j <= s; ++j) {
    c.mu[j] = (2.0 * j - 1.0) / j * bj[j] / bj[j - 1];
    c.nu[j] = -(j - 1.0) / j * bj[j] / bj[j - 2];
    c.mut[j] = 4.0 * (2.0 * j - 1.0) / (j * ss) * bj[j] / bj[j - 1];
    c.gt[j] = (bj[j - 1] - 1.0) * c.mut[j];
  }
  return c;
}

static void build_metrics(sts_grid* g) {
  const int n1 = g->n1g, n2 = g->n2, n3 = g->n3;
  const bool sph = g->geom == STS_GEOM_SPHERICAL;
  const auto& x1f = g->h_x1f;
  const auto& x1c = g->h_x1c;
  const auto& x2f = g->h_x2f;
  const auto& x2c = g->h_x2c;
  const auto& x3f = g->h_x3f;
  const auto& x3c = g->h_x3c;
  std::vector<double> F1r(n1, 0), F2r(n1), F3r(n1), Vr(n1), iH1(n1, 0), iG2(n1);
  std::vector<double> F1t(n2), F2t(n2, 0), F3t(n2), Vt(n2), iH2(n2, 0), iG3(n2);
  std::vector<double> F1p(n3), F2p(n3), F3p(n3, 0), Vp(n3), iH3(n3, 0);
  for (int i = 0; i < n1; ++i) {
    const double a = x1f[i], b = x1f[i + 1], dx = b - a;
    if (i + 1 < n1) iH1[i] = 1.0 / (x1c[i + 1] - x1c[i]);
    if (sph) {
      if (i + 1 < n1) F1r[i] = b * b * iH1[i];
      F2r[i] = F3r[i] = 0.5 * (b * b - a * a) / x1c[i];
      Vr[i] = (b * b * b - a * a * a) / 3.0;
      iG2[i] = 1.0 / x1c[i];
    } else {
      F1r[i] = iH1[i];
      F2r[i] = F3r[i] = Vr[i] = dx;
      iG2[i] = 1.0;
    }
  }
  for (int j = 0; j < n2; ++j) {
    const double a = x2f[j], b = x2f[j + 1], dy = b - a;
    if (j + 1 < n2) iH2[j] = 1.0 / (x2c[j + 1] - x2c[j]);
    if (sph) {
      F1t[j] = Vt[j] = std::cos(a) - std::cos(b);
      if (j + 1 < n2) F2t[j] = std::sin(b) * iH2[j];
      F3t[j] = dy / std::sin(x2c[j]);
      iG3[j] = 1.0 / std::sin(x2c[j]);
    } else {
      F1t[j] = F3t[j] = Vt[j] = dy;
      F2t[j] = iH2[j];
      iG3[j] = 1.0;
    }
  }
  const double period = x3f[n3] - x3f[0];
  for (int k = 0; k < n3; ++k) {
    const double dz = x3f[k + 1] - x3f[k];
    if (k + 1 < n3) iH3[k] = 1.0 / (x3c[k + 1] - x3c[k]);
    else if (g->periodic3) iH3[k] = 1.0 / (x3c[0] + period - x3c[k]);
    F1p[k] = F2p[k] = Vp[k] = dz;
    F3p[k] = iH3[k];
  }
  std::vector<const std::vector<double>*> arrs = {&F1r, &F2r, &F3r, &Vr, &iH1, &iG2, &F1t, &F2t, &F3t,
                                                   &Vt, &iH2, &iG3, &F1p, &F2p, &F3p, &Vp, &iH3};
  std::vector<double> host;
  std::vector<size_t> offs;
  for (auto* a : arrs) {
    offs.push_back(host.size());
    host.insert(host.end(), a->begin(), a->end());
  }
  // device copies of x1f, x1c for the f_c(r) profile of the face diffusivity
  offs.push_back(host.size());
  host.insert(host.end(), x1f.begin(), x1f.end());
  offs.push_back(host.size());
  host.insert(host.end(), x1c.begin(), x1c.end());
  STS_CUDA(cudaMalloc(&g->d_metrics, host.size() * sizeof(double)));
  STS_CUDA(cudaMemcpy(g->d_metrics, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice));
  const double* d = g->d_metrics;
  Metrics& m = g->m;
  m.F1r = d + offs[0]; m.F2r = d + offs[1]; m.F3r = d + offs[2]; m.Vr = d + offs[3]; m.iH1 = d + offs[4];
  m.iG2 = d + offs[5]; m.F1t = d + offs[6]; m.F2t = d + offs[7]; m.F3t = d + offs[8]; m.Vt = d + offs[9];
  m.iH2 = d + offs[10]; m.iG3 = d + offs[11]; m.F1p = d + offs[12]; m.F2p = d + offs[13]; m.F3p = d + offs[14];
  m.Vp = d + offs[15]; m.iH3 = d + offs[16];
}

static const double* d_x1f(const sts_grid* g) {
  const size_t n1 = g->n1g, n2 = g->n2, n3 = g->n3;
  return g->d_metrics + 6 * n1 + 6 * n2 + 5 * n3;
}
static const double* d_x1c(const sts_grid* g) { return d_x1f(g) + g->n1g + 1; }

// One RKL2 super-step (Fig. 2) Y0 = u0 -> u1 with frozen vertex
// coefficients `ev`; M0, A, B are NF-sized scratch fields (A, B rotate the stages).
static void rkl2_core(sts_grid* g, int mode, int ncomp, const double* u0, double* u1, const double* k1,
                      const double* k2, const double* k3, const double* bb, const double* w, double dt, int s,
                      const std::vector<const double*>& ev, double* M0, double* A, double* B, cudaStream_t st) {
  const Rkl2Coef co = rkl2_coefs(s);
  // deviation form (sts_grid_set_rkl2_deviation): D_j = Y_j - Y0 for the stages before
  // the last, where the TMA kernels take both stage forms
  bool dev = false;
  if (g->tma && g->rkl2_dev && s >= 3) {
    StencilCall c = make_call(g, g->slabs[0], mode, ncomp, EPI_RKL2_DSTAGE, A, k1, k2, k3, bb, w);
    c.ev = ev[0];
    c.ea.out = off(B, g->slabs[0]);
    c.ea.ym2 = off(B, g->slabs[0]);
    c.ea.m0 = off(M0, g->slabs[0]);
    StencilCall f = make_call(g, g->slabs[0], mode, ncomp, EPI_RKL2_FIRST, u0, k1, k2, k3, bb, w);
    f.ev = ev[0];
    f.ea.out = off(A, g->slabs[0]);
    f.ea.out2 = off(M0, g->slabs[0]);
    dev = mode == STS_MODE_ANISO ? aniso_tma_eligible(c) && aniso_tma_eligible(f)
                                 : iso_tma_eligible(c) && iso_tma_eligible(f);
  }
  // stage 1: M0 = F(Y0), Y1 = Y0 + mu~_1 dt M0 (deviation form: D1 = mu~_1 dt M0)
  sweep(g, {{H_U, u0, ncomp}}, st, [&](size_t si) {
    const Slab& sl = g->slabs[si];
    StencilCall c = make_call(g, sl, mode, ncomp, EPI_RKL2_FIRST, u0, k1, k2, k3, bb, w);
    c.ev = ev[si];
    c.ea.out = off(A, sl);
    c.ea.out2 = off(M0, sl);
    c.ea.c0 = co.mut[1] * dt;
    c.ea.a0 = dev ? 0.0 : 1.0;
    return c;
  });
  // stages 2..s (buffer rotation: Y_{j-1} (D_{j-1}) in `cur`, Y_{j-2} (D_{j-2}) in `prev`;
  // prev == nullptr stands for D_0 = 0)
  const double* prev = dev ? nullptr : u0;
  double* cur = A;
  for (int j = 2; j <= s; ++j) {
    double* dst;
    if (j == s) dst = u1;
    else if (prev == u0 || prev == nullptr) dst = B;    // never overwrite Y0
    else dst = const_cast<double*>(prev);               // in place over Y_{j-2}
    const bool dstage = dev && j < s;
    sweep(g, {{H_U, cur, ncomp}}, st, [&](size_t si) {
      const Slab& sl = g->slabs[si];
      StencilCall c = make_call(g, sl, mode, ncomp, dstage ? EPI_RKL2_DSTAGE : EPI_RKL2_STAGE, cur, k1, k2, k3, bb,
                                w);
      c.ev = ev[si];
      c.ea.out = off(dst, sl);
      c.ea.ym2 = off(prev ? prev : cur, sl);             // (D_0 = 0: nu multiplies a finite dummy)
      c.ea.y0 = off(u0, sl);
      c.ea.m0 = off(M0, sl);
      c.ea.mu = co.mu[j];
      c.ea.nu = prev ? co.nu[j] : 0.0;
      c.ea.c0 = co.mut[j] * dt;
      if (dev) {
        // D_j = mu D_{j-1} + nu D_{j-2} + mu~ dt M D_{j-1} + (mu~ + gamma~) dt M0; the last
        // stage adds Y0 back (c2 = 1)
        c.ea.c1 = (co.mut[j] + co.gt[j]) * dt;
        c.ea.c2 = 1.0;
      } else {
        c.ea.c1 = co.gt[j] * dt;
        c.ea.c2 = 1.0 - co.mu[j] - co.nu[j];
      }
      return c;
    });
    prev = cur;
    cur = dst;
  }
}

// frozen vertex coefficients of one call (ANISO): the binding's, built once per binding,
// or built into `scratch` (vertex_coef_doubles(g, mode) doubles) from the call's arrays
static std::vector<const double*> call_vertex_coefs(sts_grid* g, int mode, const Coefs& cf, double* scratch,
                                                    cudaStream_t st, cudaStream_t build_stream = nullptr) {
  if (mode != STS_MODE_ANISO) return std::vector<const double*>(g->slabs.size(), nullptr);
  if (!cf.slot) return build_vertex_coefs(g, mode, scratch, cf.k1, cf.k2, cf.k3, cf.b, st);
  CoefSlot& s = *cf.slot;
  const size_t n = vertex_coef_doubles(g, mode);
  cudaStream_t bs = build_stream ? build_stream : st;
  double* base = slot_dbuf(s, n);
  if (!s.ev_ok) {
    if (bs != st) slot_wait_readers(s, bs);   // (on the compute stream the readers are earlier)
    build_vertex_coefs(g, mode, base, cf.k1, cf.k2, cf.k3, cf.b, bs);
    s.ev_ok = true;
  }
  std::vector<const double*> out;
  size_t o = 0;
  for (auto& sl : g->slabs) {
    out.push_back(base + o);
    o += rnd(3 * (size_t)ev_cstride(sl.nl, g->n2, g->n3));
  }
  return out;
}

// scratch doubles a call needs for its vertex coefficients
static size_t call_ev_doubles(const sts_grid* g, int mode, const Coefs& cf) {
  return cf.slot ? 0 : vertex_coef_doubles(g, mode);
}

// metric-folded face coefficients K1, K2, K3 and wV of the merged isotropic PCG pass
// ([4][nl][plane] at stride Nr): the binding's (once per binding) or built into `scratch`
static double* call_premul(sts_grid* g, const Coefs& cf, double* scratch, size_t Nr, cudaStream_t st,
                           cudaStream_t build_stream = nullptr) {
  double* pre = scratch;
  if (cf.slot) {
    CoefSlot& s = *cf.slot;
    pre = slot_dbuf(s, 4 * Nr);
    if (s.pre_ok) return pre;
    if (build_stream && build_stream != st) {
      slot_wait_readers(s, build_stream);
      st = build_stream;
    }
  }
  for (auto& sl : g->slabs) {
    Timed t(g, STS_K_VERTEX_COEF, st);   // (the isotropic counterpart of the frozen vertex coefficients)
    launch_iso_premul(slab_geo(g, sl), off(cf.k1, sl), off(cf.k2, sl), off(cf.k3, sl), off(cf.w, sl), off(pre, sl),
                      off(pre + Nr, sl), off(pre + 2 * Nr, sl), off(pre + 3 * Nr, sl), st);
  }
  if (cf.slot) cf.slot->pre_ok = true;
  return pre;
}

// ----------------------------------------------------------------------------
// BE + Jacobi-PCG (Fig. 1): one solve, enqueued on `st`.
// Single-process solves with graphs enabled run the iteration loop on the device: the
// first three iterations directly, then a WHILE conditional graph node whose body is one
// iteration pair (k even, k odd: the ping-pong buffers swap back) and whose condition
// kernel continues while any component is neither converged nor stopped at kmax -- no
// host polling, so the call need not wait for the solve.  Instrumented (timing) and NCCL
// solves poll device-side convergence flags from the host in batches sized by the
// observed convergence rate.  Results (iterations, status) are published to the handle's
// mapped mailbox at the end of the solve; `done` is called with them on the host.
// ----------------------------------------------------------------------------
// destroy the loop graphs of earlier solves that have completed (all: wait for them).
// Destroying an executable graph synchronizes the device, so this runs only when many
// have accumulated (and in sts_grid_destroy).
static void reap_execs(sts_grid* g, bool all) {
  auto& v = g->retired_execs;
  for (size_t i = 0; i < v.size();) {
    const cudaError_t q = all ? cudaEventSynchronize(v[i].second) : cudaEventQuery(v[i].second);
    if (q == cudaErrorNotReady) {
      ++i;
      continue;
    }
    cudaGraphExecDestroy(v[i].first);
    cudaEventDestroy(v[i].second);
    v[i] = v.back();
    v.pop_back();
  }
  cudaGetLastError();
}

struct PcgResult {
  int iters[MAXC];
  int status;
};

static void CUDART_CB pcg_mailbox_cb(void* p);

struct PcgCallback {
  sts_grid* g;
  int ncomp;
  int* iters_out;
  int* status_out;
  long long body_launches, body_local, body_global;
};

static int mailbox_status(const PcgScal* hsc, int ncomp) {
  bool broke = false, kmax = false;
  for (int c = 0; c < ncomp; ++c) {
    broke = broke || (hsc[c].flags & PCG_BREAKDOWN);
    kmax = kmax || (hsc[c].flags & PCG_KMAX) || !hsc[c].done;
  }
  return broke ? STS_ERR_BREAKDOWN : (kmax ? STS_ERR_NOT_CONVERGED : STS_OK);
}

static void CUDART_CB pcg_mailbox_cb(void* p) {
  auto* cb = static_cast<PcgCallback*>(p);
  const auto* hsc = reinterpret_cast<const PcgScal*>(cb->g->h_pinned);
  const int bodies = reinterpret_cast<const int*>(cb->g->h_pinned + (sizeof(PcgScal) * MAXC) / sizeof(double))[0];
  if (cb->iters_out)
    for (int c = 0; c < cb->ncomp; ++c) cb->iters_out[c] = hsc[c].iters;
  if (cb->status_out) *cb->status_out = mailbox_status(hsc, cb->ncomp);
  cb->g->launches_async += bodies * cb->body_launches;
  cb->g->comm_async[0] += bodies * cb->body_local;
  cb->g->comm_async[1] += bodies * cb->body_global;
  delete cb;
}

// one BE + Jacobi-PCG solve; returns true if it ran synchronously (results already in
// the mailbox and written to iters_out / status_out)
static bool pcg_core(sts_grid* g, int mode, int ncomp, const double* un, double* un1, const Coefs& cf, double dt,
                     double rtol, int kmax, cudaStream_t st, bool write_x0, int* iters_out, int* status_out,
                     int* sync_status, bool allow_async, HostIO& io) {
  const size_t N = (size_t)g->nl * g->plane;
  const size_t NF = N * ncomp;
  const size_t NFr = rnd(NF), Nr = rnd(N);
  const double *k1 = cf.k1, *k2 = cf.k2, *k3 = cf.k3, *w = cf.w;
  const double* bb = mode == STS_MODE_ANISO ? cf.b : nullptr;
  // scratch: six [ncomp][nl][plane] fields (two-pass: r, z, y, p0, p1; merged: z0, z1,
  // w0, w1, p0, p1); d [nl][plane]; vertex coefficients (unless resident)
  // (+ the metric-folded isotropic coefficients K1, K2, K3, wV of the merged pass, unless resident)
  const bool want_pre = mode == STS_MODE_ISO && g->tma && g->pcg_merged;
  const size_t npre = (want_pre && !cf.slot) ? 4 * Nr : 0;
  const size_t evn = call_ev_doubles(g, mode, cf);
  double* base = ws_get(g, (6 * NFr + Nr + npre + evn) * sizeof(double));
  double* r = base;
  double* z = base + NFr;
  double* y = base + 2 * NFr;
  double* pb[2] = {base + 3 * NFr, base + 4 * NFr};
  double* d = base + 6 * NFr;
  double* evbase = base + 6 * NFr + Nr + npre;
  // merged iteration buffers: p_k in p4[k % 4] (the pass reads p_{k-2} and p_{k-1}, writes
  // p_k; z is never stored), w_k in wb[k % 2]; R0 leaves z0 in p4[0]
  double* p4[4] = {base, base + NFr, base + 3 * NFr, base + 4 * NFr};
  double* wb[2] = {base + 2 * NFr, base + 5 * NFr};
  double* x = un1;
  const double rtol2 = rtol * rtol;
  const long long cs = (long long)g->nl * g->plane;

  exchange_coeffs(g, mode, k1, k2, k3, bb, st);
  const auto ev = call_vertex_coefs(g, mode, cf, evbase, st);
  // the S-pass (p update + x update + A p) is ONE fused TMA kernel where eligible
  bool fused = false;
  if (g->tma) {
    StencilCall c = make_call(g, g->slabs[0], mode, ncomp, EPI_PCG_S, z, k1, k2, k3, bb, w);
    c.u2 = view(g, g->slabs[0], H_P, pb[0]);
    c.ev = ev[0];
    c.ea.out = off(y, g->slabs[0]);
    c.ea.out2 = off(pb[1], g->slabs[0]);
    c.ea.x = off(x, g->slabs[0]);
    c.u3 = view(g, g->slabs[0], H_D, d);
    fused = aniso_tma_eligible(c) || iso_tma_eligible(c);
  }
  // merged iteration (one pass + one reduction per iteration, sts_grid_set_pcg_merged);
  // eligibility does not depend on the coefficient values, so it is decided before the
  // isotropic coefficients are folded
  bool merged = false;
  double* pre = nullptr;
  if (g->tma && g->pcg_merged) {
    StencilCall c = make_call(g, g->slabs[0], mode, ncomp, EPI_PCG_M, p4[0], k1, k2, k3, bb, w);
    c.u2 = view(g, g->slabs[0], H_W, wb[0]);
    c.u3 = view(g, g->slabs[0], H_P, p4[1]);
    c.ev = ev[0];
    c.ea.out2 = off(p4[2], g->slabs[0]);
    c.ea.out3 = off(wb[1], g->slabs[0]);
    c.ea.x = off(x, g->slabs[0]);
    c.ea.dinv = off(d, g->slabs[0]);
    if (mode == STS_MODE_ISO) {
      // (any 16 B-aligned stand-in: the folded arrays are laid out like the scratch fields)
      double* probe = base;
      c.k1.p = off(probe, g->slabs[0]);
      c.k2.p = off(probe + Nr, g->slabs[0]);
      c.k3.p = off(probe + 2 * Nr, g->slabs[0]);
      c.w = off(probe + 3 * Nr, g->slabs[0]);
      c.premul = 1;
    }
    merged = (mode == STS_MODE_ISO ? want_pre && iso_tma_eligible(c) : aniso_tma_eligible(c));
  }
  if (merged && mode == STS_MODE_ISO) pre = call_premul(g, cf, base + 6 * NFr + Nr, Nr, st);
  if (merged) fused = false;
  // isotropic fused S-pass: z = r d is formed inside the stencil pass from the staged
  // r and d, so neither the initial residual pass nor the U-pass stores z
  const bool zd = fused && mode == STS_MODE_ISO;
  double* partials = nullptr;
  long long pstride = 0;
  PcgScal* sc = nullptr;
  int k_cur = 1;   // iteration whose S-pass is being built
  auto make_r0 = [&](size_t si) {
    const Slab& sl = g->slabs[si];
    StencilCall c = make_call(g, sl, mode, ncomp, EPI_PCG_R0, un, k1, k2, k3, bb, w);
    c.ev = ev[si];
    c.ea.out = merged ? off(wb[0], sl) : off(r, sl);   // (merged: r0 itself is not needed)
    c.ea.out2 = write_x0 ? off(x, sl) : nullptr;
    c.ea.out3 = merged ? off(p4[0], sl) : (zd ? nullptr : off(z, sl));
    c.ea.out4 = off(d, sl);
    c.ea.dt = dt;
    c.ea.partials = partials;
    c.ea.pstride = pstride;
    return c;
  };
  auto make_s = [&](size_t si) {   // fused S-pass (TMA)
    const Slab& sl = g->slabs[si];
    const int first = (k_cur == 1);
    StencilCall c = make_call(g, sl, mode, ncomp, EPI_PCG_S, zd ? r : z, k1, k2, k3, bb, w);
    c.u = view(g, sl, H_Z, zd ? r : z);
    c.u2 = first ? FieldV{} : view(g, sl, H_P, pb[(k_cur - 1) & 1]);
    if (zd) c.u3 = view(g, sl, H_D, d);
    c.ev = ev[si];
    c.ea.out = off(y, sl);
    c.ea.out2 = off(pb[k_cur & 1], sl);
    c.ea.x = off(x, sl);
    c.ea.first = first;
    c.ea.dt = dt;
    c.ea.partials = partials;
    c.ea.pstride = pstride;
    c.ea.sc = sc;
    return c;
  };
  auto make_m = [&](size_t si) {   // merged iteration k_cur (TMA): fields p_{k-2}, w_{k-1}, p_{k-1}
    const Slab& sl = g->slabs[si];
    const int first = (k_cur == 1);
    const int k = k_cur;
    // (first: z0 as field 0; k = 2: p_0 = z0 stands in for p_{k-2}, its coefficient beta_1 = 0)
    double* f0 = first ? p4[0] : p4[(k - 2) & 3];
    StencilCall c = make_call(g, sl, mode, ncomp, EPI_PCG_M, f0, k1, k2, k3, bb, w);
    c.u = view(g, sl, H_Z, f0);
    c.u2 = first ? FieldV{} : view(g, sl, H_W, wb[(k - 1) & 1]);
    c.u3 = first ? FieldV{} : view(g, sl, H_P, p4[(k - 1) & 3]);
    c.ev = ev[si];
    c.ea.out = nullptr;
    c.ea.out2 = off(p4[k & 3], sl);
    c.ea.out3 = off(wb[k & 1], sl);
    c.ea.x = off(x, sl);
    c.ea.dinv = off(d, sl);
    if (mode == STS_MODE_ISO) {   // metric-folded coefficients (the k1 halo planes stay raw)
      c.k1.p = off(pre, sl);
      c.k2.p = off(pre + Nr, sl);
      c.k3.p = off(pre + 2 * Nr, sl);
      c.w = off(pre + 3 * Nr, sl);
      c.premul = 1;
    }
    c.ea.first = first;
    c.ea.dt = dt;
    c.ea.partials = partials;
    c.ea.pstride = pstride;
    c.ea.sc = sc;
    return c;
  };
  auto make_ap = [&](size_t si) {  // A p of the unfused S-pass
    const Slab& sl = g->slabs[si];
    double* pnew = pb[k_cur & 1];
    StencilCall c = make_call(g, sl, mode, ncomp, EPI_PCG_AP, pnew, k1, k2, k3, bb, w);
    c.ev = ev[si];
    c.ea.out = off(y, sl);
    c.ea.dt = dt;
    c.ea.partials = partials;
    c.ea.pstride = pstride;
    c.ea.sc = sc;
    return c;
  };
  const int sb_r0 = sweep_blocks(g, true, make_r0);
  const int sb_s = merged ? sweep_blocks(g, true, make_m)
                          : (fused ? sweep_blocks(g, true, make_s) : sweep_blocks(g, true, make_ap));
  pstride = std::max(std::max(sb_r0, sb_s), PW_BLOCKS);
  // partial rows: ncomp x (2 for R0, 1 per two-pass phase, 4 for the merged pass); then
  // the sums, the per-component scalars and the loop-body counter
  const size_t nsc = (sizeof(PcgScal) * MAXC) / sizeof(double);
  const size_t red_doubles = (size_t)4 * ncomp * pstride + 16 + nsc + 8;
  ensure_red(g, red_doubles * sizeof(double));
  partials = g->d_red;
  double* sums = partials + 4 * ncomp * pstride;
  sc = reinterpret_cast<PcgScal*>(sums + 16);
  int* body_count = reinterpret_cast<int*>(sums + 16 + nsc);
  const int npub = (int)nsc + 1;   // published: the scalars of MAXC components + the body counter

  // fused final reductions (single process): the last CTA of the S-pass / U-pass sums
  // the partials and runs the scalar phase, saving two launches per iteration
  FinRed fin_s;
  fin_s.ticket = g->d_ticket;
  fin_s.sums = sums;
  fin_s.sc = sc;
  fin_s.ncomp = ncomp;
  fin_s.nq = 1;
  fin_s.phase = PH_AP;
  fin_s.rtol2 = rtol2;
  FinRed fin_u = fin_s;
  fin_u.phase = PH_RZ;
  FinRed fin_m = fin_s;
  fin_m.nq = 4;
  fin_m.phase = PH_M;
  fin_u.ntot = PW_BLOCKS;   // set to the launched grid by launch_pcg_rupdate
  auto reduce = [&](int nblocks, int nq, int phase) {
    Timed t(g, STS_K_PCG_REDUCE, st);
    if (g->comm) {
      launch_pcg_reduce(partials, pstride, nblocks, ncomp, nq, sums, PH_NONE, sc, rtol2, st, g->d_red2, g->d_ticket + 1);
      STS_NCCL(ncclAllReduce(sums, sums, (size_t)ncomp * nq, ncclDouble, ncclSum, g->comm, st));
      launch_pcg_scalar(sums, ncomp, nq, phase, sc, rtol2, st);
      g->launches += 1;
    } else {
      launch_pcg_reduce(partials, pstride, nblocks, ncomp, nq, sums, phase, sc, rtol2, st, g->d_red2, g->d_ticket + 1);
    }
  };

  launch_pcg_init(sc, ncomp, kmax, body_count, st);
  g->launches += 1;
  // r0 = b - A x0 = dt L un ; d = 1/diag(A) ; x = un ; z0 = r0 d ; r0.z0, b.P^-1 b
  reduce(sweep(g, {{H_U, un, ncomp}}, st, make_r0), 2, PH_R0);
  if (needs_halos(g)) g->comm_global += 1;
  if (zd) exchange(g, H_D, d, 1, st);   // d is fixed for the whole solve: its halo once
  // merged iteration k: ONE pass (z_k, p_k, y_k = A p_k, w_k = d y_k, x_k; partials
  // r_k.z_k, p_k.y_k, z_k.y_k, w_k.y_k) and ONE reduction (alpha_k, r_{k+1}.z_{k+1},
  // convergence, beta_{k+1}: pcg.cuh PH_M)
  auto iteration_m = [&](int k, cudaStream_t is) {
    k_cur = k;
    if (needs_halos(g)) g->comm_global += 1;
    const FinRed* fs = (g->comm || sb_s > 4096) ? nullptr : &fin_m;
    int nbs;
    if (k == 1) nbs = sweep(g, {{H_Z, p4[0], ncomp}}, is, make_m, fs);
    else
      nbs = sweep(g, {{H_Z, p4[(k - 2) & 3], ncomp}, {H_W, wb[(k - 1) & 1], ncomp}, {H_P, p4[(k - 1) & 3], ncomp}},
                  is, make_m, fs);
    if (!fs) {
      Timed t(g, STS_K_PCG_REDUCE, is);
      launch_pcg_reduce(partials, pstride, nbs, ncomp, 4, sums, g->comm ? PH_NONE : PH_M, sc, rtol2, is, g->d_red2,
                        g->d_ticket + 1);
      if (g->comm) {
        STS_NCCL(ncclAllReduce(sums, sums, (size_t)ncomp * 4, ncclDouble, ncclSum, g->comm, is));
        launch_pcg_scalar(sums, ncomp, 4, PH_M, sc, rtol2, is);
        g->launches += 1;
      }
    }
  };
  // two-pass iteration k (Fig. 1 with the x update deferred one iteration):
  //   S: p_k = z_k + beta_{k-1} p_{k-1};  x_k = x_{k-1} + alpha_{k-1} p_{k-1};  y = A p_k;  alpha_k
  //   U: r_{k+1} = r_k - alpha_k y;  z_{k+1} = r_{k+1} d;  r.z -> convergence, beta_k
  auto iteration = [&](int k, cudaStream_t is) {
    if (merged) return iteration_m(k, is);
    k_cur = k;
    if (needs_halos(g)) g->comm_global += 2;   // p.y (alpha) and r.z (beta + convergence)
    double* pold = pb[(k - 1) & 1];
    double* pnew = pb[k & 1];
    int nbs;
    if (fused) {
      // (the last CTA finishes the reduction when the pass has few CTAs; large passes
      // keep the 1024-thread reduction kernel, which sums ~1e4 partials faster)
      const FinRed* fs = (g->comm || sb_s > 4096) ? nullptr : &fin_s;
      const double* zr = zd ? r : z;
      if (k == 1) nbs = sweep(g, {{H_Z, zr, ncomp}}, is, make_s, fs);
      else nbs = sweep(g, {{H_Z, zr, ncomp}, {H_P, pold, ncomp}}, is, make_s, fs);
    } else {
      {
        Timed t(g, STS_K_PCG_PUPDATE, is);
        launch_pcg_pnew(ncomp, (long long)N, cs, pnew, z, pold, x, sc, k == 1, is);
      }
      nbs = sweep(g, {{H_U, pnew, ncomp}}, is, make_ap);
    }
    if (!(fused && !g->comm && sb_s <= 4096)) {           // else finished by the S-pass's last CTA
      Timed t(g, STS_K_PCG_REDUCE, is);
      launch_pcg_reduce(partials, pstride, nbs, ncomp, 1, sums, g->comm ? PH_NONE : PH_AP, sc, rtol2, is, g->d_red2,
                        g->d_ticket + 1);
      if (g->comm) {
        STS_NCCL(ncclAllReduce(sums, sums, (size_t)ncomp, ncclDouble, ncclSum, g->comm, is));
        launch_pcg_scalar(sums, ncomp, 1, PH_AP, sc, rtol2, is);
        g->launches += 1;
      }
    }
    int nbu;
    {
      Timed t(g, STS_K_PCG_UPDATE, is);
      nbu = launch_pcg_rupdate(ncomp, (long long)N, cs, r, zd ? nullptr : z, y, d, sc, partials, pstride,
                               g->comm ? FinRed{} : fin_u, is);
    }
    if (g->comm) {
      Timed t(g, STS_K_PCG_REDUCE, is);
      launch_pcg_reduce(partials, pstride, nbu, ncomp, 1, sums, PH_NONE, sc, rtol2, is, g->d_red2, g->d_ticket + 1);
      STS_NCCL(ncclAllReduce(sums, sums, (size_t)ncomp, ncclDouble, ncclSum, g->comm, is));
      launch_pcg_scalar(sums, ncomp, 1, PH_RZ, sc, rtol2, is);
      g->launches += 1;
    }
  };

  auto* hsc = reinterpret_cast<PcgScal*>(g->h_pinned);
  const bool device_loop = g->graphs && !g->timing && g->comm == nullptr;
  // iterations k >= 4 repeat with this period (the buffer roles): the merged iteration's
  // p buffers rotate by k % 4, the two-pass iteration's by k % 2
  const int cycle = merged ? 4 : 2;
  // (cudaGraphExecDestroy synchronizes the device: completed loop graphs are released in
  // bulk, rarely, instead of once per solve)
  if (g->retired_execs.size() >= 64) reap_execs(g, false);
  long long body_launches = 0, body_local = 0, body_global = 0;
  if (device_loop) {
    // iterations 1..3 directly (iteration 1 is its own pass variant; every kernel variant
    // then has had its one-time attribute setup outside graph capture), then the loop
    cudaStream_t is = graph_stream(g);
    STS_CUDA(cudaEventRecord(g->ev_c, st));
    STS_CUDA(cudaStreamWaitEvent(is, g->ev_c, 0));
    for (int k = 1; k <= 3; ++k) iteration(k, is);
    cudaGraph_t cg = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool capturing = false;
    try {
      STS_CUDA(cudaGraphCreate(&cg, 0));
      cudaGraphConditionalHandle h;
      STS_CUDA(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault));
      // node 1: the first evaluation of the condition
      STS_CUDA(cudaStreamBeginCaptureToGraph(is, cg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      capturing = true;
      launch_pcg_continue(h, sc, ncomp, body_count, false, is);
      capturing = false;
      STS_CUDA(cudaStreamEndCapture(is, &cg));
      size_t nn = 1;
      cudaGraphNode_t first = nullptr;
      STS_CUDA(cudaGraphGetNodes(cg, &first, &nn));
      // node 2: WHILE (condition) { iteration pair; condition }
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t loop;
      STS_CUDA(cudaGraphAddNode(&loop, cg, &first, 1, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      const long long l0 = g->launches, cl0 = g->comm_local, cg0 = g->comm_global;
      STS_CUDA(cudaStreamBeginCaptureToGraph(is, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      capturing = true;
      for (int k = 4; k < 4 + cycle; ++k) iteration(k, is);
      launch_pcg_continue(h, sc, ncomp, body_count, true, is);
      g->launches += 1;
      capturing = false;
      STS_CUDA(cudaStreamEndCapture(is, &body));
      body_launches = g->launches - l0;
      body_local = g->comm_local - cl0;
      body_global = g->comm_global - cg0;
      g->launches = l0 + 1;   // the condition node itself
      g->comm_local = cl0;
      g->comm_global = cg0;
      STS_CUDA(cudaGraphInstantiate(&exec, cg, 0));
      STS_CUDA(cudaGraphDestroy(cg));
      cg = nullptr;
      STS_CUDA(cudaGraphLaunch(exec, is));
      cudaEvent_t done = nullptr;
      STS_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      STS_CUDA(cudaEventRecord(done, is));
      g->retired_execs.push_back({exec, done});
      exec = nullptr;
    } catch (...) {
      if (capturing) {   // leave the library's stream usable: close the capture, drop the graph
        cudaGraph_t broken = nullptr;
        if (cudaStreamEndCapture(is, &broken) == cudaSuccess && broken && broken != cg) cudaGraphDestroy(broken);
      }
      if (exec) cudaGraphExecDestroy(exec);
      if (cg) cudaGraphDestroy(cg);
      cudaGetLastError();
      throw;
    }
    STS_CUDA(cudaEventRecord(g->ev_c, is));
    STS_CUDA(cudaStreamWaitEvent(st, g->ev_c, 0));
  } else {
    // host-polled loop: batches sized from the observed convergence rate so that no more
    // than ~1-2 no-op iterations (which still exchange halos and all-reduce under NCCL)
    // follow convergence
    // With an NCCL communicator (and graphs enabled, timing off) iterations k >= 4 come
    // in identical pairs replayed from ONE captured CUDA graph (NCCL send / recv and
    // all-reduce are capturable): no host launch work and minimal gaps per iteration.
    // If the capture fails the solve continues with direct launches.
    const bool pair_graph = g->comm && g->graphs && !g->timing;
    cudaStream_t is = st;
    if (pair_graph) {
      is = graph_stream(g);
      STS_CUDA(cudaEventRecord(g->ev_c, st));
      STS_CUDA(cudaStreamWaitEvent(is, g->ev_c, 0));
    }
    cudaGraphExec_t pair_exec = nullptr;
    bool pair_failed = false;
    long long pair_launches = 0, pair_local = 0, pair_global = 0;
    int launched = 0;
    int batch = 4;
    std::vector<double> rz_prev(ncomp, 0.0);
    while (true) {
      launch_publish(reinterpret_cast<const double*>(sc), npub, g->d_pinned, is);
      g->launches += 1;
      STS_CUDA(cudaStreamSynchronize(is));
      bool all_done = true;
      for (int c = 0; c < ncomp; ++c) all_done = all_done && hsc[c].done;
      if (all_done || launched >= kmax) break;
      if (launched > 0) {
        // remaining iterations ~ log(thresh / rz) / log(rate), rate per iteration from the last batch
        int need = 1;
        for (int c = 0; c < ncomp; ++c) {
          if (hsc[c].done) continue;
          const double rz = hsc[c].rz, th = hsc[c].thresh, r0 = rz_prev[c];
          int n = 64;
          if (rz > 0.0 && r0 > rz && th > 0.0) {
            const double lrate = std::log(rz / r0) / batch;
            n = (int)std::ceil(std::log(th / rz) / lrate);
          }
          need = std::max(need, std::max(1, std::min(64, n)));
        }
        batch = need;
      }
      for (int c = 0; c < ncomp; ++c) rz_prev[c] = hsc[c].rz;
      const int nb = std::min(batch, kmax - launched);
      for (int it = 0; it < nb;) {
        const int k = launched + it + 1;
        if (pair_graph && !pair_failed && k >= 4 && (k % cycle) == 0 && it + cycle <= nb) {
          if (!pair_exec) {
            const long long l0 = g->launches, cl0 = g->comm_local, cg0 = g->comm_global;
            cudaGraph_t graph = nullptr;
            bool capturing = false;
            try {
              STS_CUDA(cudaStreamBeginCapture(is, cudaStreamCaptureModeThreadLocal));
              capturing = true;
              for (int j = 0; j < cycle; ++j) iteration(k + j, is);
              capturing = false;
              STS_CUDA(cudaStreamEndCapture(is, &graph));
              STS_CUDA(cudaGraphInstantiate(&pair_exec, graph, 0));
              STS_CUDA(cudaGraphDestroy(graph));
            } catch (const Error&) {
              if (capturing) {
                cudaGraph_t broken = nullptr;
                if (cudaStreamEndCapture(is, &broken) == cudaSuccess && broken) cudaGraphDestroy(broken);
              } else if (graph) {
                cudaGraphDestroy(graph);
              }
              cudaGetLastError();
              pair_exec = nullptr;
              pair_failed = true;
            }
            pair_launches = g->launches - l0;
            pair_local = g->comm_local - cl0;
            pair_global = g->comm_global - cg0;
            g->launches = l0;
            g->comm_local = cl0;
            g->comm_global = cg0;
            if (pair_failed) continue;   // (this pair again, launched directly)
          }
          STS_CUDA(cudaGraphLaunch(pair_exec, is));
          g->launches += pair_launches;
          g->comm_local += pair_local;
          g->comm_global += pair_global;
          it += cycle;
        } else {
          iteration(k, is);
          it += 1;
        }
      }
      launched += nb;
      batch = nb;
    }
    if (pair_exec) {
      cudaEvent_t done = nullptr;
      STS_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      STS_CUDA(cudaEventRecord(done, is));
      g->retired_execs.push_back({pair_exec, done});
    }
    if (pair_graph) {
      STS_CUDA(cudaEventRecord(g->ev_c, is));
      STS_CUDA(cudaStreamWaitEvent(st, g->ev_c, 0));
    }
  }
  {
    Timed t(g, STS_K_PCG_XFINAL, st);
    // p_k in pk[k % 4] (the two-pass iteration's p ping-pongs: its pattern repeats)
    const double* pk[4] = {merged ? p4[0] : pb[0], merged ? p4[1] : pb[1], merged ? p4[2] : pb[0],
                           merged ? p4[3] : pb[1]};
    launch_pcg_xfinal(ncomp, (long long)N, cs, x, pk, sc, st);
  }
  launch_publish(reinterpret_cast<const double*>(sc), npub, g->d_pinned, st);
  g->launches += 1;
  slot_used(cf.slot, st);
  io.end();
  const bool async = allow_async && device_loop && !io.sync;
  if (async) {
    auto* cb = new PcgCallback{g, ncomp, iters_out, status_out, body_launches, body_local, body_global};
    const cudaError_t e = cudaLaunchHostFunc(st, pcg_mailbox_cb, cb);
    if (e != cudaSuccess) {
      delete cb;
      STS_CUDA(e);
    }
    return false;
  }
  STS_CUDA(cudaStreamSynchronize(st));
  const int bodies = reinterpret_cast<const int*>(g->h_pinned + nsc)[0];
  g->launches += bodies * body_launches;
  g->comm_local += bodies * body_local;
  g->comm_global += bodies * body_global;
  if (iters_out)
    for (int c = 0; c < ncomp; ++c) iters_out[c] = hsc[c].iters;
  *sync_status = mailbox_status(hsc, ncomp);
  return true;
}

}  // namespace sts

using namespace sts;

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int sts_version(void) { return 100; }

const char* sts_last_error(void) { return g_last_error.c_str(); }

int sts_grid_create(sts_grid** out, int geom, int n1, int n2, int n3, const double* x1f, const double* x1c,
                    const double* x2f, const double* x2c, const double* x3f, const double* x3c, int periodic3,
                    int i0, int nl, int n_virtual, int device) {
  return guard([&] {
    STS_REQUIRE(out != nullptr, "out is NULL");
    *out = nullptr;
    STS_REQUIRE(geom == STS_GEOM_CARTESIAN || geom == STS_GEOM_SPHERICAL, "bad geom");
    STS_REQUIRE(n1 >= 1 && n2 >= 1 && n3 >= 1, "n1, n2, n3 must be >= 1");
    STS_REQUIRE(x1f && x1c && x2f && x2c && x3f && x3c, "coordinate arrays must be non-NULL");
    STS_REQUIRE(i0 >= 0 && nl >= 1 && i0 + nl <= n1, "slab [i0, i0+nl) outside [0, n1)");
    STS_REQUIRE(n_virtual >= 1 && n_virtual <= nl, "n_virtual must be in [1, nl]");
    STS_REQUIRE(n_virtual == 1 || (i0 == 0 && nl == n1), "virtual slabs need the whole grid");
    auto mono = [](const double* f, const double* c, int n) {
      for (int i = 0; i < n; ++i)
        if (!(f[i] < f[i + 1]) || !(c[i] > f[i] && c[i] < f[i + 1])) return false;
      return true;
    };
    STS_REQUIRE(mono(x1f, x1c, n1) && mono(x2f, x2c, n2) && mono(x3f, x3c, n3),
                "faces must increase and centres lie strictly inside their cells");
    if (geom == STS_GEOM_SPHERICAL) {
      STS_REQUIRE(x1f[0] > 0.0, "spherical r must be > 0");
      STS_REQUIRE(x2f[0] >= 0.0 && x2f[n2] <= M_PI + 1e-12, "spherical theta must lie in [0, pi]");
    }
    DeviceGuard dg(device);
    auto* g = new sts_grid();
    g->comm_async[0] = 0;
    g->comm_async[1] = 0;
    g->device = device;
    g->geom = geom;
    g->n1g = n1;
    g->n2 = n2;
    g->n3 = n3;
    g->periodic3 = periodic3 ? 1 : 0;
    g->i0 = i0;
    g->nl = nl;
    g->n_virtual = n_virtual;
    g->plane = (long long)n2 * n3;
    // ncu cannot profile the kernel nodes of a graph with conditional nodes: profiling runs
    // set STS_PCG_HOST_LOOP=1 to launch the same PCG kernels from the host-polled loop
    if (const char* e = std::getenv("STS_PCG_HOST_LOOP")) g->graphs = (e[0] == '0');
    g->h_x1f.assign(x1f, x1f + n1 + 1);
    g->h_x1c.assign(x1c, x1c + n1);
    g->h_x2f.assign(x2f, x2f + n2 + 1);
    g->h_x2c.assign(x2c, x2c + n2);
    g->h_x3f.assign(x3f, x3f + n3 + 1);
    g->h_x3c.assign(x3c, x3c + n3);
    try {
      build_metrics(g);
      // slabs: contiguous, sizes differ by at most one plane
      for (int s = 0; s < n_virtual; ++s) {
        Slab sl;
        const int base = nl / n_virtual, rem = nl % n_virtual;
        sl.i0 = i0 + s * base + std::min(s, rem);
        sl.nl = base + (s < rem ? 1 : 0);
        sl.off = (long long)(sl.i0 - i0) * g->plane;
        sl.has_lo = sl.i0 > 0;        // a neighbour below exists (virtual slab or rank)
        sl.has_hi = sl.i0 + sl.nl < n1;
        g->slabs.push_back(sl);
      }
      STS_CUDA(cudaHostAlloc(&g->h_pinned, 4096, cudaHostAllocMapped));
      STS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g->d_pinned), g->h_pinned, 0));
      STS_CUDA(cudaMalloc(&g->d_ticket, 64 * sizeof(unsigned int)));
      STS_CUDA(cudaMemset(g->d_ticket, 0, 64 * sizeof(unsigned int)));
      STS_CUDA(cudaMalloc(&g->d_red2, (size_t)R2_MAXBLOCKS * 4 * MAXC * sizeof(double)));
      STS_CUDA(cudaMalloc(&g->d_gmax, 64));
    } catch (...) {
      sts_grid_destroy(g);
      throw;
    }
    *out = g;
  });
}

int sts_grid_destroy(sts_grid* g) {
  if (!g) return STS_OK;
  return guard([&] {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    for (auto& s : g->slabs) {
      for (auto* p : s.halo_lo) if (p) cudaFree(p);   // halo_hi points into the same allocation
    }
    if (g->comm) ncclCommDestroy(g->comm);
    if (g->comm_stream) cudaStreamDestroy(g->comm_stream);
    if (g->ev_a) cudaEventDestroy(g->ev_a);
    if (g->ev_b) cudaEventDestroy(g->ev_b);
    if (g->ev_c) cudaEventDestroy(g->ev_c);
    if (g->graph_stream) cudaStreamDestroy(g->graph_stream);
    for (auto& r : g->pending) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : g->free_events) cudaEventDestroy(e);
    reap_execs(g, true);
    if (g->h2d_stream || g->d2h_stream || !g->stage_pool.empty()) cudaDeviceSynchronize();
    for (auto& b : g->stage_pool) {
      cudaFree(b.p);
      cudaEventDestroy(b.ev);
    }
    g->stage_pool.clear();
    for (auto& sl : g->slot) slot_free(sl);
    if (g->h2d_stream) cudaStreamDestroy(g->h2d_stream);
    if (g->d2h_stream) cudaStreamDestroy(g->d2h_stream);
    if (g->ev_h2d_last) cudaEventDestroy(g->ev_h2d_last);
    if (g->ev_d2h_last) cudaEventDestroy(g->ev_d2h_last);
    if (g->d_metrics) cudaFree(g->d_metrics);
    if (g->ws.base) cudaFree(g->ws.base);
    if (g->d_red) cudaFree(g->d_red);
    if (g->d_ticket) cudaFree(g->d_ticket);
    if (g->d_red2) cudaFree(g->d_red2);
    if (g->d_gmax) cudaFree(g->d_gmax);
    if (g->coef_stream) cudaStreamDestroy(g->coef_stream);
    if (g->ev_coef) cudaEventDestroy(g->ev_coef);
    if (g->ev_pos) cudaEventDestroy(g->ev_pos);
    if (g->h_pinned) cudaFreeHost(g->h_pinned);
    delete g;
    if (prev >= 0) cudaSetDevice(prev);
  });
}

int sts_grid_workspace_bytes(const sts_grid* g, size_t* bytes) {
  return guard([&] {
    STS_REQUIRE(g && bytes, "NULL argument");
    size_t slots = 0;
    for (auto& s : g->slot) {
      slots += s.dbytes;
      for (int i = 0; i < 5; ++i) slots += s.own_n[i] * sizeof(double);
      for (int d = 0; d < 3; ++d)
        if (s.kfk[d]) slots += (size_t)g->nl * g->plane * sizeof(double);
    }
    *bytes = g->ws.bytes + g->red_bytes + g->halo_bytes + g->stage_bytes + slots;
  });
}

int sts_grid_kernel_launches(const sts_grid* g, long long* count) {
  return guard([&] {
    STS_REQUIRE(g && count, "NULL argument");
    *count = g->launches + g->launches_async.load();
  });
}

int sts_grid_pcg_xmodes(const sts_grid* g, int ncomp, int* skipped, int* caught_up) {
  return guard([&] {
    STS_REQUIRE(g && skipped && caught_up && ncomp >= 1 && ncomp <= MAXC, "bad arguments");
    const auto* hsc = reinterpret_cast<const PcgScal*>(g->h_pinned);
    for (int c = 0; c < ncomp; ++c) {
      skipped[c] = hsc[c].nskip;
      caught_up[c] = hsc[c].ncatch;
    }
  });
}

int sts_grid_comm_counts(const sts_grid* g, long long* local, long long* global_) {
  return guard([&] {
    STS_REQUIRE(g && local && global_, "NULL argument");
    *local = g->comm_local + g->comm_async[0].load();
    *global_ = g->comm_global + g->comm_async[1].load();
  });
}

int sts_grid_set_timing(sts_grid* g, int enable) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    g->timing = enable != 0;
  });
}

int sts_grid_set_graphs(sts_grid* g, int enable) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    g->graphs = enable != 0;
  });
}

int sts_grid_set_pcg_merged(sts_grid* g, int enable) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    g->pcg_merged = enable != 0;
  });
}

int sts_grid_set_halo_overlap(sts_grid* g, int enable) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    g->halo_overlap = enable != 0;
  });
}

int sts_grid_set_rkl2_deviation(sts_grid* g, int enable) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    g->rkl2_dev = enable != 0;
  });
}

int sts_grid_set_tma(sts_grid* g, int enable) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    g->tma = enable != 0;
  });
}

int sts_grid_timing_reset(sts_grid* g) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    DeviceGuard dg(g->device);
    collect_timing(g);
    for (int k = 0; k < STS_K_NCLASSES; ++k) {
      g->acc_ms[k] = 0.0;
      g->acc_n[k] = 0;
    }
  });
}

int sts_grid_timing(sts_grid* g, int kind, long long* count, double* ms) {
  return guard([&] {
    STS_REQUIRE(g && count && ms, "NULL argument");
    STS_REQUIRE(kind >= 0 && kind < STS_K_NCLASSES, "bad kernel class");
    DeviceGuard dg(g->device);
    collect_timing(g);
    *count = g->acc_n[kind];
    *ms = g->acc_ms[kind];
  });
}

int sts_nccl_unique_id(void* out, size_t nbytes) {
  return guard([&] {
    STS_REQUIRE(out && nbytes >= sizeof(ncclUniqueId), "buffer too small for an ncclUniqueId");
    ncclUniqueId id;
    STS_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

int sts_comm_init(sts_grid* g, int nranks, int rank, const void* uid, size_t nbytes) {
  return guard([&] {
    STS_REQUIRE(g && uid && nbytes >= sizeof(ncclUniqueId), "bad arguments");
    STS_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    STS_REQUIRE(g->n_virtual == 1, "virtual slabs and NCCL ranks cannot be combined");
    STS_REQUIRE(g->comm == nullptr, "communicator already initialised");
    STS_REQUIRE((rank == 0) == (g->i0 == 0) && (rank == nranks - 1) == (g->i0 + g->nl == g->n1g),
                "rank order must match r-slab order");
    DeviceGuard dg(g->device);
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    g->nranks = nranks;
    g->rank = rank;
    // (a 1-rank communicator is created too: the NCCL reduction path then runs on one GPU)
    STS_NCCL(ncclCommInitRank(&g->comm, nranks, id, rank));
    comm_stream(g);
  });
}

int sts_face_kappa_spitzer(sts_grid* g, const double* T, double* k1, double* k2, double* k3, double kappa0,
                           double T_cut, double fc_r0, double fc_w, void* stream) {
  return guard([&] {
    STS_REQUIRE(g && T, "NULL argument");
    const bool resident = !k1 && !k2 && !k3;
    STS_REQUIRE(resident || (k1 && k2 && k3), "k1, k2, k3 must all be given (or all NULL: resident output)");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)g->nl * g->plane;
    CoefSlot& s = g->slot[slot_index(STS_MODE_ANISO)];
    if (resident) {
      for (int d = 0; d < 3; ++d)
        if (!s.kfk[d]) s.kfk[d] = dev_alloc(N, "resident face diffusivities");
      k1 = s.kfk[0];
      k2 = s.kfk[1];
      k3 = s.kfk[2];
    }
    // a resident output on a single-slab grid is computed on the coefficient stream: it
    // waits only for its input (the upload of a host T, the caller's stream for a device
    // T) and for the last readers of the binding it overwrites
    const bool on_cs = resident && !needs_halos(g);
    const bool dev_T = is_device_ptr(T);
    const cudaStream_t cst = st;
    if (on_cs) {
      st = coef_stream(g);
      slot_wait_readers(s, st);
      if (dev_T) {
        STS_CUDA(cudaEventRecord(g->ev_pos, cst));
        STS_CUDA(cudaStreamWaitEvent(st, g->ev_pos, 0));
      }
    }
    HostIO io(g, st);
    io.input(T, N);
    io.output(k1, N);
    io.output(k2, N);
    io.output(k3, N);
    io.begin();
    exchange(g, H_AUX, T, 1, st);
    Slab whole;
    whole.i0 = g->i0;
    whole.nl = g->nl;
    whole.off = 0;
    Geo G = slab_geo(g, whole);
    FieldV Tv;
    Tv.p = T;
    // with a real neighbour above, the last plane's r-face uses the received halo
    Tv.hi = (g->comm && g->slabs[0].has_hi) ? g->slabs[0].halo_hi[H_AUX] : nullptr;
    {
      Timed t(g, STS_K_FACE_KAPPA, st);
      launch_face_kappa(G, Tv, k1, k2, k3, kappa0, T_cut, fc_r0, fc_w, d_x1f(g), d_x1c(g), st);
    }
    io.end();
    if (on_cs) {   // later work on the caller's stream sees the new diffusivities
      STS_CUDA(cudaEventRecord(g->ev_coef, st));
      STS_CUDA(cudaStreamWaitEvent(cst, g->ev_coef, 0));
    }
    if (resident) {   // bind them (b and w of the binding are kept)
      for (int d = 0; d < 3; ++d) s.k[d] = s.kfk[d];
      s.bound = true;
      slot_invalidate(s);
      slot_update_user_dev(s);
    }
  });
}

int sts_grid_bind_coeffs(sts_grid* g, int mode, const double* k1, const double* k2, const double* k3,
                         const double* b, const double* w, void* stream) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    STS_REQUIRE(mode == STS_MODE_ISO || mode == STS_MODE_ANISO, "mode must be STS_MODE_ISO or STS_MODE_ANISO");
    STS_REQUIRE(mode == STS_MODE_ANISO || !b, "b is bound for STS_MODE_ANISO only");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)g->nl * g->plane;
    CoefSlot& s = g->slot[slot_index(mode)];
    const double* src[5] = {k1, k2, k3, b, w};
    const size_t cnt[5] = {N, N, N, 3 * N, N};
    const double** dst[5] = {&s.k[0], &s.k[1], &s.k[2], &s.b, &s.w};
    bool uploaded = false;
    for (int i = 0; i < 5; ++i) {
      if (!src[i]) continue;
      const Mem kind = mem_kind(src[i]);
      if (kind == Mem::Device) {
        *dst[i] = src[i];
        continue;
      }
      // host array: into the library-owned copy, once the binding's last readers (calls on
      // the compute stream, binding work on the coefficient stream) have run
      if (s.own_n[i] < cnt[i]) {
        if (s.own[i]) STS_CUDA(cudaFree(s.own[i]));
        s.own[i] = nullptr;
        s.own[i] = dev_alloc(cnt[i], "resident coefficients");
        s.own_n[i] = cnt[i];
      }
      cudaStream_t cs = copy_stream(g, true);
      slot_wait_readers(s, cs);
      if (g->coef_stream) STS_CUDA(cudaStreamWaitEvent(cs, g->ev_coef, 0));
      STS_CUDA(cudaMemcpyAsync(s.own[i], src[i], cnt[i] * sizeof(double), cudaMemcpyHostToDevice, cs));
      if (kind == Mem::Pageable) STS_CUDA(cudaStreamSynchronize(cs));
      *dst[i] = s.own[i];
      uploaded = true;
    }
    if (uploaded) {
      STS_CUDA(cudaEventRecord(g->ev_h2d_last, g->h2d_stream));
      STS_CUDA(cudaStreamWaitEvent(st, g->ev_h2d_last, 0));
      g->h2d_used = true;
    }
    s.bound = true;
    slot_invalidate(s);
    slot_update_user_dev(s);
  });
}

int sts_grid_unbind_coeffs(sts_grid* g, int mode) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    STS_REQUIRE(mode == STS_MODE_ISO || mode == STS_MODE_ANISO, "mode must be STS_MODE_ISO or STS_MODE_ANISO");
    DeviceGuard dg(g->device);
    STS_CUDA(cudaDeviceSynchronize());   // enqueued work may still read the binding
    slot_free(g->slot[slot_index(mode)]);
  });
}

int sts_grid_join(sts_grid* g, void* stream) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (g->h2d_used) STS_CUDA(cudaStreamWaitEvent(st, g->ev_h2d_last, 0));
    if (g->d2h_used) STS_CUDA(cudaStreamWaitEvent(st, g->ev_d2h_last, 0));
  });
}

int sts_grid_synchronize(sts_grid* g) {
  return guard([&] {
    STS_REQUIRE(g, "NULL grid");
    DeviceGuard dg(g->device);
    for (cudaStream_t s : {g->h2d_stream, g->d2h_stream, g->graph_stream, g->comm_stream})
      if (s) STS_CUDA(cudaStreamSynchronize(s));
  });
}

int sts_op_apply(sts_grid* g, int mode, int ncomp, const double* u, double* out, const double* k1,
                 const double* k2, const double* k3, const double* b, const double* w, void* stream) {
  return guard([&] {
    STS_REQUIRE(g && u && out, "NULL argument");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)g->nl * g->plane;
    HostIO io(g, st);
    Coefs cf;
    resolve_coefs(cf, g, mode, k1, k2, k3, b, w, io, N);
    check_mode(mode, ncomp, cf.b);
    STS_REQUIRE((const void*)u != (const void*)out, "u and out must not alias");
    io.input(u, N * ncomp);
    io.output(out, N * ncomp);
    io.begin();
    double* base = ws_get(g, (call_ev_doubles(g, mode, cf) + 1) * sizeof(double));
    exchange_coeffs(g, mode, cf.k1, cf.k2, cf.k3, cf.b, st);
    const auto ev = call_vertex_coefs(g, mode, cf, base, st);
    sweep(g, {{H_U, u, ncomp}}, st, [&](size_t si) {
      const Slab& s = g->slabs[si];
      StencilCall c = make_call(g, s, mode, ncomp, EPI_F, u, cf.k1, cf.k2, cf.k3, cf.b, cf.w);
      c.ev = ev[si];
      c.ea.out = off(out, s);
      return c;
    });
    slot_used(cf.slot, st);
    io.end();
  });
}

int sts_dt_euler(sts_grid* g, int mode, const double* k1, const double* k2, const double* k3, const double* b,
                 const double* w, double* dt_out, void* stream) {
  return guard([&] {
    STS_REQUIRE(g && dt_out, "NULL argument");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)g->nl * g->plane;
    HostIO io(g, st);
    Coefs cf;
    resolve_coefs(cf, g, mode, k1, k2, k3, b, w, io, N);
    check_mode(mode, 1, cf.b);
    double lam = cf.slot ? cf.slot->lam : -1.0;
    if (lam < 0.0) {   // (resident coefficients: computed once per binding)
      // Resident coefficients on a single-slab grid: the binding's work (vertex /
      // folded coefficients into the other generation, the Gershgorin pass) runs on the
      // coefficient stream, which waits only for the binding's uploads (and the caller's
      // stream if a bound array is the caller's) -- so the host gets dt_exp while the
      // previous binding's solves still compute.  Otherwise on the caller's stream.
      const bool on_cs = cf.slot && !needs_halos(g) && !g->comm;
      const cudaStream_t cst = st;
      if (on_cs) {
        st = coef_stream(g);
        if (cf.slot->user_dev) {
          STS_CUDA(cudaEventRecord(g->ev_pos, cst));
          STS_CUDA(cudaStreamWaitEvent(st, g->ev_pos, 0));
        }
        if (g->h2d_used) STS_CUDA(cudaStreamWaitEvent(st, g->ev_h2d_last, 0));
      }
      io.st = st;
      io.begin();
      exchange_coeffs(g, mode, cf.k1, cf.k2, cf.k3, cf.b, st);
      // ANISO: the row sums come from the frozen vertex coefficients (the binding's are
      // then ready for the advance that follows)
      double* scratch = on_cs ? nullptr : ws_get(g, (call_ev_doubles(g, mode, cf) + 1) * sizeof(double));
      const auto ev = call_vertex_coefs(g, mode, cf, scratch, cst, st);
      auto* dmax = reinterpret_cast<unsigned long long*>(g->d_gmax);
      STS_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st));
      for (size_t si = 0; si < g->slabs.size(); ++si) {
        StencilCall c = make_call(g, g->slabs[si], mode, 1, 0, nullptr, cf.k1, cf.k2, cf.k3, cf.b, cf.w);
        c.ev = ev[si];
        Timed t(g, mode == STS_MODE_ANISO ? STS_K_ANISO_GERSH : STS_K_ISO_GERSH, st);
        launch_gershgorin(c, dmax, st);
      }
      if (g->comm) STS_NCCL(ncclAllReduce(g->d_gmax, g->d_gmax, 1, ncclDouble, ncclMax, g->comm, st));
      // (the isotropic binding's folded coefficients of the merged PCG pass, while here)
      if (on_cs && mode == STS_MODE_ISO && g->tma && g->pcg_merged)
        call_premul(g, cf, nullptr, rnd((size_t)g->nl * g->plane), cst, st);
      launch_publish(g->d_gmax, 1, g->d_pinned + DT_MAILBOX, st);
      g->launches += 1;
      io.end();
      if (on_cs) {
        STS_CUDA(cudaEventRecord(g->ev_coef, st));
        STS_CUDA(cudaStreamWaitEvent(cst, g->ev_coef, 0));
        STS_CUDA(cudaEventSynchronize(g->ev_coef));
      } else {
        slot_used(cf.slot, st);
        STS_CUDA(cudaStreamSynchronize(st));
      }
      lam = g->h_pinned[DT_MAILBOX];
      if (cf.slot) cf.slot->lam = lam;
    }
    *dt_out = lam > 0.0 ? 2.0 / lam : std::numeric_limits<double>::infinity();
  });
}

int rkl2_num_stages(double dt, double dt_exp, int force_odd) {
  if (!(std::isfinite(dt) && std::isfinite(dt_exp)) || dt < 0.0 || dt_exp <= 0.0) {
    set_error("rkl2_num_stages: need finite dt >= 0 and dt_exp > 0");
    return STS_ERR_ARG;
  }
  const double ratio = dt / dt_exp;
  const double x = std::ceil((std::sqrt(9.0 + 16.0 * ratio) - 1.0) / 2.0);
  if (x > 1e8) {
    set_error("rkl2_num_stages: stage count overflow");
    return STS_ERR_ARG;
  }
  int s = std::max(2, (int)x);
  if (force_odd && (s % 2 == 0)) s += 1;
  return s;
}

int rkl2_advance(sts_grid* g, int mode, int ncomp, const double* u0, double* u1, const double* k1,
                 const double* k2, const double* k3, const double* b, const double* w, double dt, int s,
                 void* stream) {
  return guard([&] {
    STS_REQUIRE(g && u0 && u1, "NULL argument");
    STS_REQUIRE(s >= 2, "s must be >= 2");
    STS_REQUIRE(std::isfinite(dt) && dt >= 0.0, "dt must be finite and >= 0");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)g->nl * g->plane;
    const size_t NF = N * ncomp;
    HostIO io(g, st);
    Coefs cf;
    resolve_coefs(cf, g, mode, k1, k2, k3, b, w, io, N);
    check_mode(mode, ncomp, cf.b);
    io.input(u0, NF);
    // host arrays (even an in-place u0 == u1) are staged separately: the result goes to
    // its own device buffer and back; a device in-place advance is safe because Y0 is
    // only read pointwise after stage 1
    io.output(u1, NF);
    io.begin();
    const size_t NFr = rnd(NF);
    double* base = ws_get(g, (3 * NFr + call_ev_doubles(g, mode, cf)) * sizeof(double));
    exchange_coeffs(g, mode, cf.k1, cf.k2, cf.k3, cf.b, st);
    const auto ev = call_vertex_coefs(g, mode, cf, base + 3 * NFr, st);
    rkl2_core(g, mode, ncomp, u0, u1, cf.k1, cf.k2, cf.k3, cf.b, cf.w, dt, s, ev, base, base + NFr, base + 2 * NFr,
              st);
    slot_used(cf.slot, st);
    io.end();
  });
}

int rkl2_advance_hybrid(sts_grid* g, int mode, int ncomp, const double* u0, double* u1, const double* k1,
                        const double* k2, const double* k3, const double* b, const double* w, double dt,
                        double dt_exp, double euler_frac, int n_euler, int n_sub, int* stages_out, void* stream) {
  return guard([&] {
    STS_REQUIRE(g && u0 && u1, "NULL argument");
    STS_REQUIRE(std::isfinite(dt) && dt >= 0.0 && std::isfinite(dt_exp) && dt_exp > 0.0, "bad dt / dt_exp");
    STS_REQUIRE(euler_frac >= 0.0 && euler_frac < 1.0, "euler_frac must be in [0, 1)");
    STS_REQUIRE(n_sub >= 1, "n_sub must be >= 1");
    if (n_euler < 0)   // default (DESIGN R11): sub-steps of dt_exp/2, which annihilate the highest mode
      n_euler = euler_frac == 0.0 ? 0 : (int)std::ceil(euler_frac * dt / (0.5 * dt_exp) - 1e-12);
    STS_REQUIRE((n_euler == 0) == (euler_frac == 0.0), "n_euler > 0 exactly when euler_frac > 0");
    const double dte = n_euler ? euler_frac * dt / n_euler : 0.0;
    STS_REQUIRE(dte <= dt_exp * (1.0 + 1e-12), "explicit Euler sub-step exceeds dt_exp");
    const double dtr = (1.0 - euler_frac) * dt / n_sub;
    const int s = rkl2_num_stages(dtr, dt_exp, 0);
    STS_REQUIRE(s >= 2, "stage count");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)g->nl * g->plane;
    const size_t NF = N * ncomp;
    HostIO io(g, st);
    Coefs cf;
    resolve_coefs(cf, g, mode, k1, k2, k3, b, w, io, N);
    check_mode(mode, ncomp, cf.b);
    io.input(u0, NF);
    io.output(u1, NF);
    io.begin();
    const size_t NFr = rnd(NF);
    // scratch: M0, A, B (RKL2 stages), E0, E1 (sub-step ping-pong), vertex coefficients
    double* base = ws_get(g, (5 * NFr + call_ev_doubles(g, mode, cf)) * sizeof(double));
    double* E[2] = {base + 3 * NFr, base + 4 * NFr};
    const double* bb = cf.b;
    exchange_coeffs(g, mode, cf.k1, cf.k2, cf.k3, bb, st);
    const auto ev = call_vertex_coefs(g, mode, cf, base + 5 * NFr, st);
    // explicit Euler prefix: u <- u + dte F(u), n_euler times
    const double* cur = u0;
    int e = 0;
    for (int i = 0; i < n_euler; ++i) {
      double* dst = E[e];
      e ^= 1;
      sweep(g, {{H_U, cur, ncomp}}, st, [&](size_t si) {
        const Slab& sl = g->slabs[si];
        StencilCall c = make_call(g, sl, mode, ncomp, EPI_RKL2_FIRST, cur, cf.k1, cf.k2, cf.k3, bb, cf.w);
        c.ev = ev[si];
        c.ea.out = off(dst, sl);
        c.ea.out2 = off(base, sl);   // F(u) (unused scratch)
        c.ea.c0 = dte;
        return c;
      });
      cur = dst;
    }
    // the remainder as n_sub RKL2 super-steps (RKL2 sub-cycling)
    for (int m = 1; m <= n_sub; ++m) {
      double* dst = (m == n_sub) ? u1 : E[e];
      if (m < n_sub) e ^= 1;
      rkl2_core(g, mode, ncomp, cur, dst, cf.k1, cf.k2, cf.k3, bb, cf.w, dtr, s, ev, base, base + NFr, base + 2 * NFr,
                st);
      cur = dst;
    }
    if (stages_out) {
      stages_out[0] = n_euler;
      stages_out[1] = s;
    }
    slot_used(cf.slot, st);
    io.end();
  });
}

static int pcg_entry(sts_grid* g, int mode, int ncomp, const double* un, double* un1, const double* k1,
                     const double* k2, const double* k3, const double* b, const double* w, double dt, double rtol,
                     int kmax, int* iters_out, int* status_out, void* stream, bool allow_async) {
  int status = STS_OK;
  bool synchronous = true;
  int rc = guard([&] {
    STS_REQUIRE(g && un && un1, "NULL argument");
    STS_REQUIRE(kmax >= 1, "kmax must be >= 1");
    STS_REQUIRE(std::isfinite(dt) && dt >= 0.0 && std::isfinite(rtol) && rtol >= 0.0, "bad dt / rtol");
    DeviceGuard dg(g->device);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)g->nl * g->plane;
    const size_t NF = N * ncomp;
    HostIO io(g, st);
    Coefs cf;
    resolve_coefs(cf, g, mode, k1, k2, k3, b, w, io, N);
    check_mode(mode, ncomp, cf.b);
    const bool alias = (const void*)un == (const void*)un1;
    // same DEVICE array for un and un1: x0 is already in place; otherwise write it
    const bool write_x0 = !(alias && is_device_ptr(un1));
    io.input(un, NF);
    io.output(un1, NF);
    io.begin();
    synchronous = pcg_core(g, mode, ncomp, un, un1, cf, dt, rtol, kmax, st, write_x0, iters_out, status_out,
                           &status, allow_async, io);
  });
  if (rc != STS_OK) return rc;
  if (!synchronous) return STS_OK;   // results arrive with the stream (status_out)
  if (status_out) *status_out = status;
  if (status == STS_ERR_BREAKDOWN)
    set_error("be_pcg_solve: PCG breakdown (p.A p <= 0 or a non-finite scalar: A not SPD or non-finite input)");
  else if (status == STS_ERR_NOT_CONVERGED)
    set_error("be_pcg_solve: kmax reached before convergence");
  return status;
}

int be_pcg_solve(sts_grid* g, int mode, int ncomp, const double* un, double* un1, const double* k1,
                 const double* k2, const double* k3, const double* b, const double* w, double dt, double rtol,
                 int kmax, int* iters_out, void* stream) {
  return pcg_entry(g, mode, ncomp, un, un1, k1, k2, k3, b, w, dt, rtol, kmax, iters_out, nullptr, stream, false);
}

int be_pcg_solve_async(sts_grid* g, int mode, int ncomp, const double* un, double* un1, const double* k1,
                       const double* k2, const double* k3, const double* b, const double* w, double dt, double rtol,
                       int kmax, int* iters_out, int* status_out, void* stream) {
  return pcg_entry(g, mode, ncomp, un, un1, k1, k2, k3, b, w, dt, rtol, kmax, iters_out, status_out, stream, true);
}

}  // extern "C"
