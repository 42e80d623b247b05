// fz_api.cu -- the C ABI of libfz (include/fz.h): validation, workspace carving, launch
// sequences, host<->device control-block round trips, status mapping.
#include <nvtx3/nvToolsExt.h>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "fz_launch.h"

namespace fz {
static thread_local int t_launches = 0;

// ---- per-kernel CUDA-event profiling (tracing) ----
namespace {
struct ProfRec {
    int id;
    cudaEvent_t a, b;
    bool done;   // end event recorded (set by ~LaunchProf under g_prof_mu)
};
std::mutex g_prof_mu;
bool g_prof_on = false;
uint64_t g_prof_mask = ~0ull;     // kernels recorded (bit = KernelId)
std::vector<ProfRec*> g_prof_pending;   // heap records: stable while the vector grows
std::vector<cudaEvent_t> g_prof_pool;
double g_prof_ms[K_COUNT];
int g_prof_n[K_COUNT];

cudaEvent_t prof_event()
{
    if (!g_prof_pool.empty()) {
        cudaEvent_t e = g_prof_pool.back();
        g_prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

static std::atomic<int> g_variant{0};
int variant_bits() { return g_variant.load(std::memory_order_relaxed); }
void set_variant_bits(int v) { g_variant.store(v, std::memory_order_relaxed); }

LaunchProf::LaunchProf(KernelId id_, cudaStream_t st_) : id(id_), st(st_), slot(-1)
{
    ++t_launches;
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (!g_prof_on || !((g_prof_mask >> id) & 1)) return;
    ProfRec* r = new ProfRec{id, prof_event(), prof_event(), false};
    cudaEventRecord(r->a, st);
    g_prof_pending.push_back(r);
    rec = r;     // the record itself, not an index: another thread's fz_profile_read may
    slot = 1;    // compact the pending vector meanwhile (it skips records not yet done)
}

LaunchProf::~LaunchProf()
{
    if (slot < 0) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    ProfRec* r = static_cast<ProfRec*>(rec);
    cudaEventRecord(r->b, st);
    r->done = true;
}
}  // namespace fz

using namespace fz;

static thread_local char g_cuda_err[256] = "";
static thread_local int g_last_launches = 0;
static thread_local uint8_t g_last_hdr[128];
static thread_local bool g_have_hdr = false;

namespace {

// variant bits for A/B timing (128: unfused y scan in the decoder), fz_debug_set_variant
int exp_bits() { return fz::variant_bits(); }

// Per public call: launch accounting and an NVTX range named after the entry point (tracing:
// visible in Nsight Systems / ncu --nvtx; header-only NVTX 3, a no-op without a tool attached).
struct LaunchScope {
    explicit LaunchScope(const char* name) { fz::t_launches = 0; nvtxRangePushA(name); }
    ~LaunchScope() { g_last_launches = fz::t_launches; nvtxRangePop(); }
};

fz_status cuda_fail(cudaError_t e)
{
    snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return FZ_ERR_CUDA;
}

#define FZ_CUDA(call)                                \
    do {                                             \
        cudaError_t e_ = (call);                     \
        if (e_ != cudaSuccess) return cuda_fail(e_); \
    } while (0)

bool shape_n(const fz_shape* s, uint64_t* n)
{
    if (s == nullptr || s->ndim < 1 || s->ndim > 3) return false;
    uint64_t m = 1;
    for (uint32_t k = 0; k < s->ndim; ++k) {
        if (s->dims[k] == 0 || s->dims[k] > 0xFFFFFFFFull) return false;
        m *= s->dims[k];
        if (m > 0xFFFFFFFFull) return false;   // element indices are u32 (R16)
    }
    *n = m;
    return true;
}

Geom geom_of(const fz_shape& s, uint64_t n)
{
    Geom g{};
    g.n = (uint32_t)n;
    g.ndim = s.ndim;
    if (s.ndim == 1) { g.nx = (uint32_t)n; g.P = (uint32_t)n; }
    else if (s.ndim == 2) { g.nx = (uint32_t)s.dims[1]; g.P = (uint32_t)n; }
    else { g.nx = (uint32_t)s.dims[2]; g.P = (uint32_t)(s.dims[1] * s.dims[2]); }
    return g;
}

uint64_t tiles_of(uint64_t n) { return (n + kTileCodes - 1) / kTileCodes; }

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// f3: bytes of the log field kept after the compress workspace's sections (FZ_EB_PWREL)
size_t log_field_bytes(uint64_t n) { return (size_t)((4 * n + 255) & ~255ull); }

struct Work {
    Layout L;
    uint8_t* base;
    Ctrl* ctrl() const { return reinterpret_cast<Ctrl*>(base + L.ctrl); }
    unsigned long long* status() const { return reinterpret_cast<unsigned long long*>(base + L.status); }
    uint2* ocnt() const { return reinterpret_cast<uint2*>(base + L.ocnt); }
    uint2* obase() const { return reinterpret_cast<uint2*>(base + L.obase); }
    uint2* opre() const { return reinterpret_cast<uint2*>(base + L.opre); }
    uint2* dstage() const { return reinterpret_cast<uint2*>(base + L.dstage); }
    uint2* vstage() const { return reinterpret_cast<uint2*>(base + L.vstage); }
    uint4* tstage() const { return L.tstage ? reinterpret_cast<uint4*>(base + L.tstage) : nullptr; }
    uint32_t* zloc() const { return reinterpret_cast<uint32_t*>(base + L.zloc); }
    uint32_t* zbsum() const { return reinterpret_cast<uint32_t*>(base + L.zbsum); }
};

bool zb_layout(const fz_shape& s)
{
    return s.ndim == 3 && zb_shape(3, s.dims[1], s.dims[2], s.dims[0]);
}

// the compress workspace of a shape: z-band / row-walker staging, or the row-codes path's
// code field and masks (2-D and 3-D shapes whose planes are not whole tiles)
Layout layout_of(const fz_shape& s, uint64_t n, uint64_t T)
{
    const bool zb = zb_layout(s);
    return compress_layout(n, T, zb, !zb && rc_layout_shape(s));
}

// f1 chunk-local Lorenzo: 3-D fields whose tiles hold whole rows of one plane;
// chunk = 16 planes x one tile (2048 / nx rows).  Header word: cz | cy << 16.
constexpr uint32_t kClDepth = 16;
bool cl_shape(const fz_shape& s)
{
    return zb_layout(s) && s.dims[2] <= (uint64_t)kTileCodes && kTileCodes % s.dims[2] == 0;
}
uint32_t cl_chunk(const fz_shape& s)
{
    return kClDepth | (uint32_t)(kTileCodes / s.dims[2]) << 16;
}
// a slab of a chunk-local field: whole chunks of planes (the last one may end at nz)
bool cl_slab(const fz_shape& s, uint64_t n, uint64_t tb, uint64_t te)
{
    if (!cl_shape(s)) return false;
    const uint64_t tpp = s.dims[1] * s.dims[2] / kTileCodes, T = tiles_of(n);
    return tb % (tpp * kClDepth) == 0 && (te == T || te % (tpp * kClDepth) == 0);
}

CompressArgs make_args(const Work& W, const float* field, uint64_t base, const Geom& g,
                       uint32_t tb, uint32_t te)
{
    CompressArgs a{};
    a.field = field;
    a.base = base;
    a.g = g;
    a.tile_begin = tb;
    a.tile_end = te;
    a.dstage = W.dstage();
    a.vstage = W.vstage();
    a.dcap = W.L.dcap;
    a.vcap = W.L.vcap;
    a.status = W.status();
    a.ocnt = W.ocnt();
    a.obase = W.obase();
    a.opre = W.opre();
    a.ctrl = W.ctrl();
    a.tstage = W.tstage();
    if (W.L.rcodes) {
        a.rc_codes = reinterpret_cast<uint16_t*>(W.base + W.L.rcodes);
        a.rc_vmask = reinterpret_cast<uint32_t*>(W.base + W.L.rmask);
        a.rc_dmask = a.rc_vmask + rc_mask_words(W.L.ntiles);
    }
    return a;
}

fz_status err_status(int32_t e)
{
    if (e == kErrStall) {
        snprintf(g_cuda_err, sizeof g_cuda_err, "look-back watchdog fired (device-side stall)");
        return FZ_ERR_CUDA;
    }
    return (fz_status)e;
}

fz_status read_ctrl(const Work& W, Ctrl* h, cudaStream_t st)
{
    FZ_CUDA(cudaMemcpyAsync(h, W.ctrl(), sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    FZ_CUDA(cudaStreamSynchronize(st));
    return FZ_OK;
}

// Where the outlier records of a compressed range go (records or split lists).
struct OutDest {
    uint2* drec = nullptr;
    uint2* vrec = nullptr;
    uint32_t* didx = nullptr;
    int32_t* dval = nullptr;
    uint32_t* vidx = nullptr;
    uint32_t* vbits = nullptr;
};

// Phase 1: init (+ range + params on the device) -> fused kernel -> totals (+ header).
fz_status compress_run(const Work& W, const CompressArgs& a, const fz_params* hp, int mode, double eb,
                       uint8_t* hdr_out, uint64_t out_cap, const fz_shape& s, uint64_t n, Ctrl* h,
                       cudaStream_t st, const float* log_src = nullptr)
{
    const uint32_t tb = a.tile_begin, nt = a.tile_end - a.tile_begin;
    // status words are per scan unit, indexed from the range start; outlier counts per tile
    FZ_CUDA(launch_init(W.ctrl(), W.status(), W.ocnt() + tb, nt, hp, st, a.cl ? cl_chunk(s) : 0u));
    // f3 (FZ_EB_PWREL): a.field is the log field y = log32(x) in the workspace (R25)
    if (log_src != nullptr) FZ_CUDA(launch_log_fwd(log_src, const_cast<float*>(a.field), n, W.ctrl(), st));
    const bool zr = compress_uses_zr(a);
    if (a.cl && !zr && !compress_uses_zb(a)) return FZ_ERR_ARG;
    if (!zr && !compress_uses_zb(a) && compress_uses_rc(a)) {
        // row-codes two-pass path: pass A (row walk -> code field + outlier masks), pass B
        // (tiles in stream order -> flags + staged blocks + outlier records), then the same
        // popcount scan, compaction and finalize as the z-band path
        if (hp == nullptr) FZ_CUDA(launch_range(a.field, n, W.ctrl(), st));
        CompressArgs b = a;
        b.derive = hp == nullptr;
        b.eb_mode = mode;
        b.eb = eb;
        b.n_hdr = n;
        FZ_CUDA(launch_compress_rc(b, st));
        const uint32_t T = a.tile_end - a.tile_begin;
        FZ_CUDA(launch_tile_offsets(a.flags_out, T, W.zloc(), W.zbsum(), W.ctrl(), st, ~1ull));
        FZ_CUDA(launch_compact(a.flags_out, W.zloc(), W.zbsum(), W.tstage(), a.payload_out, a.payload_cap, T,
                               hdr_out, out_cap, s, n, tiles_of(n), W.ctrl(), st));
        if (h == nullptr) return FZ_OK;
        return read_ctrl(W, h, st);
    }
    if (zr || compress_uses_zb(a)) {
        // z-band two-pass compressor: pass 1 derives the parameters in its prologue, writes
        // the flags and stages each tile's blocks; the popcount scan of the flags gives the
        // offsets, k_compact moves the blocks, k_finalize writes totals + header
        // C0 fused into the row walker's first phase when it walks the whole field
        // (variant bit 2097152: separate k_range launch, for A/B)
        const bool fuse = zr && hp == nullptr && a.base == 0 && a.tile_begin == 0 && a.tile_end == tiles_of(n) &&
                          !(exp_bits() & 2097152);
        if (hp == nullptr && !fuse) FZ_CUDA(launch_range(a.field, n, W.ctrl(), st));
        CompressArgs b = a;
        b.derive = hp == nullptr;
        b.fuse_range = fuse ? ((exp_bits() & 4194304) ? 2u : 1u) : 0u;
        b.eb_mode = mode;
        b.eb = eb;
        b.n_hdr = n;
        FZ_CUDA(zr ? launch_compress_zr(b, st) : launch_compress_zb(b, st));
        const uint32_t T = a.tile_end - a.tile_begin;
        FZ_CUDA(launch_tile_offsets(a.flags_out, T, W.zloc(), W.zbsum(), W.ctrl(), st, ~1ull));
        FZ_CUDA(launch_compact(a.flags_out, W.zloc(), W.zbsum(), W.tstage(), a.payload_out, a.payload_cap, T,
                               hdr_out, out_cap, s, n, tiles_of(n), W.ctrl(), st));
        if (h == nullptr) return FZ_OK;
        return read_ctrl(W, h, st);
    }
    // the warp-specialized kernel derives the parameters in its prologue and its last CTA
    // writes totals + header, so k_params and k_finalize are not launched for it
    const bool fused = compress_uses_ws(a);
    if (hp == nullptr) {
        FZ_CUDA(launch_range(a.field, n, W.ctrl(), st));
        if (!fused) FZ_CUDA(launch_params(W.ctrl(), mode, eb, n, st));
    }
    CompressArgs b = a;
    if (fused) {
        b.derive = hp == nullptr;
        b.finalize = 1;
        b.eb_mode = mode;
        b.eb = eb;
        b.hdr_out = hdr_out;
        b.hdr_cap = out_cap;
        b.ndim = s.ndim;
        for (uint32_t k = 0; k < 3; ++k) b.dims[k] = k < s.ndim ? s.dims[k] : 1;
        b.n_hdr = n;
        b.T_hdr = tiles_of(n);
    }
    FZ_CUDA(launch_compress(b, st));
    if (!fused) FZ_CUDA(launch_finalize(hdr_out, out_cap, s, n, tiles_of(n), W.ctrl(), st));
    if (h == nullptr) return FZ_OK;    // asynchronous: the caller reads ctrl later
    return read_ctrl(W, h, st);
}

// Phase 2 (only when outliers exist): per-tile exclusive offsets, then either a copy of
// the staged records or -- when the staging area overflowed -- a rescan of the tiles that
// writes the records straight to their final places.
fz_status place_outliers(const Work& W, CompressArgs a, const Ctrl& h, const OutDest& d, cudaStream_t st)
{
    if (h.nd + h.nv == 0) return FZ_OK;
    const uint32_t tb = a.tile_begin, nt = a.tile_end - a.tile_begin;
    FZ_CUDA(launch_outlier_scan(W.ocnt() + tb, W.opre() + tb, nt, st));
    if (h.stage_overflow && a.cl) return FZ_ERR_WORKSPACE;   // the rescan kernels are field-global only
    if (!h.stage_overflow) {
        FZ_CUDA(launch_outlier_place(W.ocnt() + tb, W.obase() + tb, W.opre() + tb, nt, W.dstage(), W.vstage(),
                                     d.drec, d.vrec, d.didx, d.dval, d.vidx, d.vbits, st));
    } else {
        FZ_CUDA(cudaMemsetAsync(&W.ctrl()->ticket, 0, sizeof(uint32_t), st));
        a.rescan = 1;
        a.dstage = d.drec;
        a.vstage = d.vrec;
        a.o_didx = d.didx;
        a.o_dval = d.dval;
        a.o_vidx = d.vidx;
        a.o_vbits = d.vbits;
        a.dcap = h.nd;
        a.vcap = h.nv;
        FZ_CUDA(launch_compress(a, st));
    }
    FZ_CUDA(cudaStreamSynchronize(st));
    return FZ_OK;
}

void write_header_host(uint8_t* h, const fz_shape& s, uint64_t n, uint64_t T, const fz_params& p,
                       const fz_counts& c, uint64_t total, uint32_t chunk = 0)
{
    memset(h, 0, 128);
    memcpy(h, "FZB2", 4);
    const uint16_t ver = 1,
                   fl = (uint16_t)((p.mode == FZ_EB_REL ? 1u : 0u) | (p.fallback ? 2u : 0u) | (chunk ? 4u : 0u) |
                                   (p.mode == FZ_EB_PWREL ? 8u : 0u));
    memcpy(h + 4, &ver, 2);
    memcpy(h + 6, &fl, 2);
    h[8] = (uint8_t)s.ndim;
    memcpy(h + 10, &chunk, 4);
    for (uint32_t k = 0; k < 3; ++k) {
        uint64_t d = k < s.ndim ? s.dims[k] : 1;
        memcpy(h + 16 + 8 * k, &d, 8);
    }
    memcpy(h + 40, &n, 8);
    memcpy(h + 48, &p.eb_input, 8);
    memcpy(h + 56, &p.eb_abs, 8);
    memcpy(h + 64, &p.w, 4);
    memcpy(h + 68, &p.r, 4);
    memcpy(h + 72, &p.mn, 4);
    memcpy(h + 76, &p.mx, 4);
    uint64_t cnt[5] = {T, c.nnz, c.n_delta, c.n_value, total};
    memcpy(h + 80, cnt, 40);
}

fz_status compress_impl(const float* d_field, const fz_shape* s, const fz_params* hp, int mode,
                        double eb, void* d_out, size_t out_cap, size_t* out_size, void* d_work,
                        size_t work_bytes, cudaStream_t st)
{
    uint64_t n;
    if (!shape_n(s, &n) || d_field == nullptr || d_out == nullptr || out_size == nullptr ||
        d_work == nullptr || !aligned16(d_field) || !aligned16(d_out) || !aligned16(d_work))
        return FZ_ERR_ARG;
    const bool cl = (mode & FZ_CHUNK_LOCAL) != 0;
    mode &= ~FZ_CHUNK_LOCAL;
    if (cl && !cl_shape(*s)) return FZ_ERR_ARG;
    if (hp == nullptr && (!(eb > 0.0) || !std::isfinite(eb) ||
                          (mode != FZ_EB_ABS && mode != FZ_EB_REL && mode != FZ_EB_PWREL) ||
                          (mode == FZ_EB_PWREL && !(eb < 1.0))))
        return FZ_ERR_ARG;
    const bool pw = (hp ? (int)(hp->mode & ~FZ_CHUNK_LOCAL) : mode) == FZ_EB_PWREL;
    if (pw && cl) return FZ_ERR_ARG;
    const uint64_t T = tiles_of(n);
    Work W{layout_of(*s, n, T), static_cast<uint8_t*>(d_work)};
    if (work_bytes < W.L.total + (pw ? log_field_bytes(n) : 0)) return FZ_ERR_WORKSPACE;
    const Geom g = geom_of(*s, n);
    uint8_t* out = static_cast<uint8_t*>(d_out);
    // f3: the pipeline compresses y = log32(x), kept after the workspace's other sections
    const float* src = pw ? reinterpret_cast<const float*>(W.base + W.L.total) : d_field;

    CompressArgs a = make_args(W, src, 0, g, 0, (uint32_t)T);
    a.cl = cl ? 1u : 0u;
    const uint64_t fbase = kHeaderBytes, pbase = kHeaderBytes + 32 * T;
    a.flags_out = out + fbase;
    a.flags_cap = out_cap > fbase ? out_cap - fbase : 0;
    a.payload_out = out + pbase;
    a.payload_cap = out_cap > pbase ? out_cap - pbase : 0;
    Ctrl h;
    fz_status rs = compress_run(W, a, hp, mode, eb, out, out_cap, *s, n, &h, st, pw ? d_field : nullptr);
    if (rs != FZ_OK) return rs;
    if (h.err != 0) return err_status(h.err);
    *out_size = (size_t)h.total;
    if (h.total > out_cap) return FZ_ERR_CAPACITY;
    OutDest d;
    d.drec = reinterpret_cast<uint2*>(out + pbase + 16 * h.nnz);
    d.vrec = reinterpret_cast<uint2*>(out + pbase + 16 * h.nnz + 8 * h.nd);
    rs = place_outliers(W, a, h, d, st);
    if (rs == FZ_OK) {
        // the same bytes k_finalize wrote to the stream's header
        write_header_host(g_last_hdr, *s, n, T, h.p, fz_counts{h.nnz, h.nd, h.nv}, h.total,
                          cl ? cl_chunk(*s) : 0u);
        g_have_hdr = true;
    }
    return rs;
}

}  // namespace

extern "C" {

size_t fz_compress_bound(const fz_shape* s)
{
    uint64_t n;
    if (!shape_n(s, &n)) return 0;
    const uint64_t T = tiles_of(n);
    return (size_t)(kHeaderBytes + 32 * T + 4096 * T + 16 * n);
}

size_t fz_workspace_bytes(const fz_shape* s)
{
    uint64_t n;
    if (!shape_n(s, &n)) return 0;
    return layout_of(*s, n, tiles_of(n)).total;
}

size_t fz_workspace_bytes_mode(const fz_shape* s, int eb_mode)
{
    uint64_t n;
    if (!shape_n(s, &n)) return 0;
    const size_t base = layout_of(*s, n, tiles_of(n)).total;
    return (eb_mode & ~FZ_CHUNK_LOCAL) == FZ_EB_PWREL ? base + log_field_bytes(n) : base;
}

size_t fz_debug_workspace_bytes(const fz_shape* s)
{
    uint64_t n;
    if (!shape_n(s, &n)) return 0;
    const uint64_t T = tiles_of(n);
    return layout_of(*s, n, T).total + 32 * T + 4096 * T;
}

size_t fz_decompress_workspace_bytes(const fz_shape* s)
{
    uint64_t n;
    if (!shape_n(s, &n)) return 0;
    return decode_layout(*s).total;
}

fz_status fz_derive_params(float mn, float mx, int eb_mode, double eb, fz_params* p)
{
    if (p == nullptr) return FZ_ERR_ARG;
    return (fz_status)derive_params(mn, mx, eb_mode, eb, p);
}

fz_status fz_compress(const float* d_field, const fz_shape* s, int eb_mode, double eb, void* d_out,
                      size_t out_cap, size_t* out_size, void* d_work, size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    return compress_impl(d_field, s, nullptr, eb_mode, eb, d_out, out_cap, out_size, d_work,
                         work_bytes, static_cast<cudaStream_t>(stream));
}

fz_status fz_compress_with_params(const float* d_field, const fz_shape* s, const fz_params* p,
                                  void* d_out, size_t out_cap, size_t* out_size, void* d_work,
                                  size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    if (p == nullptr || !(p->w >= 1.17549435e-38f) || !std::isfinite(p->w)) return FZ_ERR_ARG;
    // the chunk-local bit selects the Lorenzo variant; the params proper (and so the header's
    // REL bit, which k_finalize derives from p.mode) never carry it
    fz_params pm = *p;
    pm.mode &= ~(uint32_t)FZ_CHUNK_LOCAL;
    return compress_impl(d_field, s, &pm, (int)p->mode, p->eb_input, d_out, out_cap, out_size, d_work,
                         work_bytes, static_cast<cudaStream_t>(stream));
}

fz_status fz_peek_header(const void* h_hdr, size_t nbytes, fz_info* info)
{
    if (h_hdr == nullptr || info == nullptr || nbytes < kHeaderBytes) return FZ_ERR_ARG;
    const uint8_t* h = static_cast<const uint8_t*>(h_hdr);
    fz_info I{};
    if (memcmp(h, "FZB2", 4) != 0) return FZ_ERR_CORRUPT;
    uint16_t ver, fl;
    memcpy(&ver, h + 4, 2);
    memcpy(&fl, h + 6, 2);
    if (ver != 1) return FZ_ERR_CORRUPT;
    I.version = ver;
    I.flags = fl;
    I.shape.ndim = h[8];
    if (I.shape.ndim < 1 || I.shape.ndim > 3) return FZ_ERR_CORRUPT;
    for (int k = 0; k < 3; ++k) memcpy(&I.shape.dims[k], h + 16 + 8 * k, 8);
    for (uint32_t k = I.shape.ndim; k < 3; ++k) {
        if (I.shape.dims[k] != 1) return FZ_ERR_CORRUPT;
        I.shape.dims[k] = 0;
    }
    uint64_t n;
    if (!shape_n(&I.shape, &n)) return FZ_ERR_CORRUPT;
    for (uint32_t k = I.shape.ndim; k < 3; ++k) I.shape.dims[k] = 1;
    memcpy(&I.n, h + 40, 8);
    if (I.n != n) return FZ_ERR_CORRUPT;
    memcpy(&I.params.eb_input, h + 48, 8);
    memcpy(&I.params.eb_abs, h + 56, 8);
    memcpy(&I.params.w, h + 64, 4);
    memcpy(&I.params.r, h + 68, 4);
    memcpy(&I.params.mn, h + 72, 4);
    memcpy(&I.params.mx, h + 76, 4);
    {
        // f1 chunk-local streams (bit 2) carry nonzero chunk dims at bytes 10-13; other
        // streams keep those bytes zero
        uint16_t cz, cy;
        memcpy(&cz, h + 10, 2);
        memcpy(&cy, h + 12, 2);
        if ((fl & 4u) ? (cz == 0 || cy == 0) : (cz != 0 || cy != 0)) return FZ_ERR_CORRUPT;
    }
    if ((fl & 1u) && (fl & 8u)) return FZ_ERR_CORRUPT;   // REL and the f3 log transform exclude each other
    I.params.mode = (fl & 8u) ? FZ_EB_PWREL : ((fl & 1u) ? FZ_EB_REL : FZ_EB_ABS);
    I.params.fallback = (fl & 2u) ? 1u : 0u;
    if (!(I.params.w > 0.0f) || !std::isfinite(I.params.w)) return FZ_ERR_CORRUPT;
    uint64_t cnt[5];
    memcpy(cnt, h + 80, 40);
    I.tiles = cnt[0];
    I.counts.nnz = cnt[1];
    I.counts.n_delta = cnt[2];
    I.counts.n_value = cnt[3];
    I.total_size = cnt[4];
    if (I.tiles != tiles_of(n)) return FZ_ERR_CORRUPT;
    if (I.counts.nnz > I.tiles * kTileBlocks || I.counts.n_delta > n || I.counts.n_value > n)
        return FZ_ERR_CORRUPT;
    if (I.total_size != kHeaderBytes + 32 * I.tiles + 16 * I.counts.nnz + 8 * I.counts.n_delta +
                            8 * I.counts.n_value)
        return FZ_ERR_CORRUPT;
    *info = I;
    return FZ_OK;
}

}  // extern "C"

namespace {

// dev_shape != nullptr: device-driven decode.  The host uses only the caller's shape (launch
// configuration); k_decode_hdr parses the stream header on the device and every kernel takes
// the section counts and the bin width from ctrl, so nothing waits for the host.
fz_status decompress_impl(const void* d_in, size_t in_size, float* d_field, int32_t* d_q, uint64_t n,
                          void* d_work, size_t work_bytes, cudaStream_t st, const void* h_hdr = nullptr,
                          bool async = false, const fz_shape* dev_shape = nullptr)
{
    if (d_in == nullptr || (d_field == nullptr && d_q == nullptr) || d_work == nullptr ||
        !aligned16(d_in) || !aligned16(d_work) || in_size < kHeaderBytes)
        return FZ_ERR_ARG;
    const bool dev = dev_shape != nullptr;
    fz_info I{};
    uint32_t chunk = 0;      // f1 chunk-local stream: cz | cy << 16 from header bytes 10-13
    if (dev) {
        uint64_t nn;
        if (!shape_n(dev_shape, &nn) || nn != n) return FZ_ERR_ARG;
        I.shape = *dev_shape;
        I.n = n;
        I.tiles = tiles_of(n);
    } else {
        uint8_t hdr[128];
        if (h_hdr != nullptr) {
            memcpy(hdr, h_hdr, 128);
        } else {
            FZ_CUDA(cudaMemcpyAsync(hdr, d_in, 128, cudaMemcpyDeviceToHost, st));
            FZ_CUDA(cudaStreamSynchronize(st));
        }
        fz_status rs = fz_peek_header(hdr, 128, &I);
        if (rs != FZ_OK) return rs;
        if (I.n != n) return FZ_ERR_ARG;
        if (I.flags & 4u) memcpy(&chunk, hdr + 10, 4);
        if (in_size < I.total_size) return FZ_ERR_CORRUPT;
    }
    const DecodeLayout L = decode_layout(I.shape);
    if (work_bytes < L.total) return FZ_ERR_WORKSPACE;
    uint8_t* wb = static_cast<uint8_t*>(d_work);
    Ctrl* ctrl = reinterpret_cast<Ctrl*>(wb + L.ctrl);
    auto* loc = reinterpret_cast<uint32_t*>(wb + L.loc);
    auto* bsum = reinterpret_cast<uint32_t*>(wb + L.bsum);
    auto* xagg = reinterpret_cast<uint2*>(wb + L.xagg);
    auto* xloc = reinterpret_cast<uint2*>(wb + L.xloc);
    auto* xbagg = reinterpret_cast<uint2*>(wb + L.xbagg);
    auto* sums = reinterpret_cast<uint32_t*>(wb + L.sums);
    const uint8_t* in = static_cast<const uint8_t*>(d_in);
    const uint64_t T = I.tiles;
    const uint64_t pbase = kHeaderBytes + 32 * T, dbase = pbase + 16 * I.counts.nnz,
                   vbase = dbase + 8 * I.counts.n_delta;
    const uint2* drec = reinterpret_cast<const uint2*>(in + dbase);
    const uint2* vrec = reinterpret_cast<const uint2*>(in + vbase);
    const Geom g = geom_of(I.shape, n);
    int32_t* q = d_q ? d_q : reinterpret_cast<int32_t*>(d_field);
    const bool deq = d_q == nullptr;

    // f1 chunk-local stream (header bit 2): one-pass chunk decode
    if (chunk != 0 && (!cl_shape(I.shape) || (chunk >> 16) != kTileCodes / I.shape.dims[2] || (chunk & 0xFFFFu) == 0))
        return FZ_ERR_ARG;   // a chunk geometry this decoder does not implement
    const bool fuse_y = chunk == 0 && decode_fuses_y(I.shape) && !(exp_bits() & 128);
    auto* drange = reinterpret_cast<uint32_t*>(wb + L.drange);
    const float* wp = (dev && deq) ? &ctrl->dec_w : nullptr;   // device bin width (dev mode)
    if (dev) {
        FZ_CUDA(launch_decode_hdr(ctrl, in, in_size, I.shape, n, T, st));
        // the popcount scan's launch also validates the outlier lists and records the per-tile
        // delta ranges (both need only the parsed header)
        FZ_CUDA(launch_tile_offsets(in + kHeaderBytes, (uint32_t)T, loc, bsum, ctrl, st, ~0ull, in + pbase, n,
                                    drange));
    } else {
        FZ_CUDA(launch_decode_init(ctrl, st));
        FZ_CUDA(launch_validate_outliers(drec, I.counts.n_delta, n, ctrl, st));
        FZ_CUDA(launch_validate_outliers(vrec, I.counts.n_value, n, ctrl, st));
        FZ_CUDA(launch_tile_offsets(in + kHeaderBytes, (uint32_t)T, loc, bsum, ctrl, st, I.counts.nnz));
        FZ_CUDA(launch_record_tiles(drec, I.counts.n_delta, (uint32_t)T, 0, drange, st));
    }
    DecodeArgs a{};
    a.flags = in + kHeaderBytes;
    a.payload = in + pbase;
    a.drec = drec;
    a.nnz_total = I.counts.nnz;
    a.nd = I.counts.n_delta;
    a.dev = dev ? 1 : 0;
    a.wp = wp;
    a.g = g;
    a.tiles = (uint32_t)T;
    a.w = deq ? I.params.w : 0.0f;
    a.q_out = q;
    a.loc = loc;
    a.bpre = bsum;
    a.xagg = xagg;
    a.ctrl = ctrl;
    a.drange = drange;
    if (fuse_y) {
        a.tpp = (uint32_t)(I.shape.dims[1] * I.shape.dims[2] / kTileCodes);
        // two CTAs per plane unless the planes alone fill the GPU several times over
        // several CTAs per plane (shorter tile chains) unless the planes alone fill the GPU
        a.yseg = 1;
        if (I.shape.dims[0] < 4 * 148 && !(exp_bits() & 512)) {
            const uint32_t want = (exp_bits() & 4096) ? 2u : kMaxYseg;
            for (uint32_t y = want; y >= 2; y /= 2)
                if (a.tpp % y == 0) { a.yseg = y; break; }
        }
        a.ycarry = reinterpret_cast<int32_t*>(wb + L.ycarry);
    }
    if (chunk != 0) {
        a.w = deq ? I.params.w : 0.0f;
        FZ_CUDA(launch_decode_cl(a, chunk & 0xFFFFu, st));
        if (deq) FZ_CUDA(launch_value_patch(d_field, vrec, I.counts.n_value, n, st));
        if (deq && (I.flags & 8u)) FZ_CUDA(launch_exp_inv(d_field, n, nullptr, st));
        if (async) return FZ_OK;
        Ctrl hc;
        FZ_CUDA(cudaMemcpyAsync(&hc, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
        FZ_CUDA(cudaStreamSynchronize(st));
        if (hc.err != 0) return err_status(hc.err);
        if (hc.nnz != I.counts.nnz) return FZ_ERR_CORRUPT;
        return FZ_OK;
    }
    if (I.shape.ndim == 1 && !(exp_bits() & 32768)) {
        // 1-D: tile sums, their scan, the decode with the carries -- no int32 field
        DzrArgs z{};
        z.flags = a.flags;
        z.payload = a.payload;
        z.drec = a.drec;
        z.nnz_total = a.nnz_total;
        z.nd = a.nd;
        z.dev = a.dev;
        z.wp = a.wp;
        z.w = a.w;
        z.ctrl = ctrl;
        z.loc = loc;
        z.bpre = bsum;
        z.drange = drange;
        z.q_out = q;
        z.ntiles = (uint32_t)T;
        // (f3's exp as its own pass here: fused into the decode it cost occupancy -- FP64
        // latency chains at 148 registers -- and ran slower than the separate pass)
        z.logt = 0;
        uint32_t* tsum = reinterpret_cast<uint32_t*>(xagg);
        FZ_CUDA(launch_decode_1d(z, n, tsum, tsum + T, reinterpret_cast<uint32_t*>(xbagg), st));
        if (deq) {
            if (dev) {
                FZ_CUDA(launch_patch_exp_dev(d_field, in + pbase, ctrl, n, st));
            } else {
                FZ_CUDA(launch_value_patch(d_field, vrec, I.counts.n_value, n, st));
                if (I.flags & 8u) FZ_CUDA(launch_exp_inv(d_field, n, nullptr, st));
            }
        }
        if (async) return FZ_OK;
        Ctrl h1;
        FZ_CUDA(cudaMemcpyAsync(&h1, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
        FZ_CUDA(cudaStreamSynchronize(st));
        if (h1.err != 0) return err_status(h1.err);
        if (!dev && h1.nnz != I.counts.nnz) return FZ_ERR_CORRUPT;
        return FZ_OK;
    }
    const bool dzr = decode_uses_dzr(I.shape), dzg = !dzr && decode_uses_dzg(I.shape);
    if ((dzr || dzg) && !(exp_bits() & 32768)) {
        // row-walking decoders: no int32 intermediate field (fz_dzr.cu; fz_dzg.cu for rows
        // that do not tile, through an un-shuffled code field)
        const DzrLayout Z = dzr ? dzr_layout(I.shape) : dzg_layout(I.shape);
        DzrArgs z{};
        z.flags = a.flags;
        z.payload = a.payload;
        z.drec = a.drec;
        z.nnz_total = a.nnz_total;
        z.nd = a.nd;
        z.dev = a.dev;
        z.wp = a.wp;
        z.w = a.w;
        z.ctrl = ctrl;
        z.loc = loc;
        z.bpre = bsum;
        z.drange = drange;
        z.q_out = q;
        z.nx = (uint32_t)I.shape.dims[2];
        z.nz = (uint32_t)I.shape.dims[0];
        z.P = (uint32_t)(I.shape.dims[1] * I.shape.dims[2]);
        z.tpp = z.P / kTileCodes;
        z.nbands = Z.nbands;
        z.nchunks = Z.nchunks;
        z.cdelta = reinterpret_cast<int32_t*>(wb + L.dzr_cdelta);
        z.dsum = reinterpret_cast<int32_t*>(wb + L.dzr_dsum);
        z.cd = reinterpret_cast<int32_t*>(wb + L.dzr_cd);
        z.ny = (uint32_t)I.shape.dims[1];
        z.cz = Z.cz;
        z.ntiles = (uint32_t)T;
        if (dzg) z.codes = reinterpret_cast<uint16_t*>(wb + L.dzg_codes);
        // f3 (header flag bit 3): exp32 fused into the dequantization and the value patch when
        // the host knows the flag; device-parsed, a separate pass checks it
        z.logt = (deq && !dev && (I.flags & 8u)) ? 1 : 0;
        FZ_CUDA(dzr ? launch_decode_dzr(z, st) : launch_decode_dzg(z, st));
        if (deq) {
            if (dev) {
                FZ_CUDA(launch_patch_exp_dev(d_field, in + pbase, ctrl, n, st));
            } else {
                FZ_CUDA(launch_value_patch(d_field, vrec, I.counts.n_value, n, st, 0, z.logt));
            }
        }
        if (async) return FZ_OK;
        Ctrl hz;
        FZ_CUDA(cudaMemcpyAsync(&hz, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
        FZ_CUDA(cudaStreamSynchronize(st));
        if (hz.err != 0) return err_status(hz.err);
        if (!dev && hz.nnz != I.counts.nnz) return FZ_ERR_CORRUPT;
        return FZ_OK;
    }
    FZ_CUDA(launch_decode_tiles(a, st, fuse_y));
    // x carries exist when some tile starts inside a row (always for 1-D fields)
    const bool carries = T > 1 && (g.ndim == 1 || !(g.nx <= kTileCodes && kTileCodes % g.nx == 0));
    if (g.ndim == 1 && !deq) { a.w = 0.0f; a.wp = nullptr; }
    if (g.ndim == 1 && !deq) {
        if (carries) FZ_CUDA(launch_xcarry(a, xloc, xbagg, true, st));
    } else {
        FZ_CUDA(launch_xcarry(a, xloc, xbagg, carries, st));
    }
    const float wq = deq ? I.params.w : 0.0f;
    if (I.shape.ndim == 2) {
        if (!fuse_y) FZ_CUDA(launch_scan_axis(q, 1, I.shape.dims[0], I.shape.dims[1], sums, wq, st, wp));
    } else if (I.shape.ndim == 3) {
        if (!fuse_y)
            FZ_CUDA(launch_scan_axis(q, I.shape.dims[0], I.shape.dims[1], I.shape.dims[2], sums, 0.0f, st));
        if (fuse_y && a.yseg >= 2)
            FZ_CUDA(launch_zwalk_ycarry(q, I.shape.dims[0], I.shape.dims[1] * I.shape.dims[2], wq, a.ycarry,
                                        (uint32_t)I.shape.dims[2], a.yseg, st, wp));
        else
            FZ_CUDA(launch_scan_axis(q, 1, I.shape.dims[0], I.shape.dims[1] * I.shape.dims[2], sums, wq, st, wp));
    }
    if (deq) {
        if (dev) {
            FZ_CUDA(launch_patch_exp_dev(d_field, in + pbase, ctrl, n, st));
        } else {
            FZ_CUDA(launch_value_patch(d_field, vrec, I.counts.n_value, n, st));
            if (I.flags & 8u) FZ_CUDA(launch_exp_inv(d_field, n, nullptr, st));
        }
    }
    if (async) return FZ_OK;     // status later: fz_decompress_result
    Ctrl h;
    FZ_CUDA(cudaMemcpyAsync(&h, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    FZ_CUDA(cudaStreamSynchronize(st));
    if (h.err != 0) return err_status(h.err);
    if (!dev && h.nnz != I.counts.nnz) return FZ_ERR_CORRUPT;   // sum of popcount(flags) == nnz
    return FZ_OK;
}

}  // namespace

extern "C" {

fz_status fz_decompress(const void* d_in, size_t in_size, float* d_field, uint64_t n, void* d_work,
                        size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    if (d_field == nullptr || !aligned16(d_field)) return FZ_ERR_ARG;
    return decompress_impl(d_in, in_size, d_field, nullptr, n, d_work, work_bytes,
                           static_cast<cudaStream_t>(stream));
}

fz_status fz_decompress_hdr(const void* d_in, size_t in_size, const void* h_hdr, float* d_field, uint64_t n,
                            void* d_work, size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    if (d_field == nullptr || !aligned16(d_field) || h_hdr == nullptr) return FZ_ERR_ARG;
    return decompress_impl(d_in, in_size, d_field, nullptr, n, d_work, work_bytes,
                           static_cast<cudaStream_t>(stream), h_hdr);
}

fz_status fz_compress_async(const float* d_field, const fz_shape* s, int eb_mode, double eb, void* d_out,
                            size_t out_cap, void* d_work, size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    uint64_t n;
    if (!shape_n(s, &n) || d_field == nullptr || d_out == nullptr || d_work == nullptr || !aligned16(d_field) ||
        !aligned16(d_out) || !aligned16(d_work))
        return FZ_ERR_ARG;
    const bool cl = (eb_mode & FZ_CHUNK_LOCAL) != 0;
    eb_mode &= ~FZ_CHUNK_LOCAL;
    if (cl && !cl_shape(*s)) return FZ_ERR_ARG;
    if (!(eb > 0.0) || !std::isfinite(eb) || (eb_mode != FZ_EB_ABS && eb_mode != FZ_EB_REL && eb_mode != FZ_EB_PWREL) ||
        (eb_mode == FZ_EB_PWREL && (cl || !(eb < 1.0))))
        return FZ_ERR_ARG;
    const bool pw = eb_mode == FZ_EB_PWREL;
    const uint64_t T = tiles_of(n);
    Work W{layout_of(*s, n, T), static_cast<uint8_t*>(d_work)};
    if (work_bytes < W.L.total + (pw ? log_field_bytes(n) : 0)) return FZ_ERR_WORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Geom g = geom_of(*s, n);
    uint8_t* out = static_cast<uint8_t*>(d_out);
    const float* src = pw ? reinterpret_cast<const float*>(W.base + W.L.total) : d_field;
    CompressArgs a = make_args(W, src, 0, g, 0, (uint32_t)T);
    a.cl = cl ? 1u : 0u;
    const uint64_t pbase = kHeaderBytes + 32 * T;
    a.flags_out = out + kHeaderBytes;
    a.flags_cap = out_cap > kHeaderBytes ? out_cap - kHeaderBytes : 0;
    a.payload_out = out + pbase;
    a.payload_cap = out_cap > pbase ? out_cap - pbase : 0;
    fz_status rs = compress_run(W, a, nullptr, eb_mode, eb, out, out_cap, *s, n, nullptr, st, pw ? d_field : nullptr);
    if (rs != FZ_OK) return rs;
    FZ_CUDA(launch_outlier_scan(W.ocnt(), W.opre(), (uint32_t)T, st, W.ctrl()));
    FZ_CUDA(launch_outlier_place_dev(W.ocnt(), W.obase(), W.opre(), (uint32_t)T, W.dstage(), W.vstage(),
                                     a.payload_out, a.payload_cap, W.ctrl(), st));
    return FZ_OK;
}

fz_status fz_compress_result(const void* d_work, size_t out_cap, size_t* out_size, void* stream)
{
    if (d_work == nullptr || out_size == nullptr) return FZ_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Ctrl h;
    FZ_CUDA(cudaMemcpyAsync(&h, d_work, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));   // compress ctrl at offset 0
    FZ_CUDA(cudaStreamSynchronize(st));
    if (h.err != 0) return err_status(h.err);
    *out_size = (size_t)h.total;
    if (h.total > out_cap) return FZ_ERR_CAPACITY;
    return FZ_OK;
}

fz_status fz_decompress_hdr_async(const void* d_in, size_t in_size, const void* h_hdr, float* d_field, uint64_t n,
                                  void* d_work, size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    if (d_field == nullptr || !aligned16(d_field) || h_hdr == nullptr) return FZ_ERR_ARG;
    return decompress_impl(d_in, in_size, d_field, nullptr, n, d_work, work_bytes,
                           static_cast<cudaStream_t>(stream), h_hdr, true);
}

fz_status fz_decompress_async(const void* d_in, size_t in_size, const fz_shape* s, float* d_field, void* d_work,
                              size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    uint64_t n;
    if (d_field == nullptr || !aligned16(d_field) || !shape_n(s, &n)) return FZ_ERR_ARG;
    return decompress_impl(d_in, in_size, d_field, nullptr, n, d_work, work_bytes,
                           static_cast<cudaStream_t>(stream), nullptr, true, s);
}

fz_status fz_decompress_result(const void* d_work, void* stream)
{
    if (d_work == nullptr) return FZ_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Ctrl h;
    FZ_CUDA(cudaMemcpyAsync(&h, d_work, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));   // decode ctrl at offset 0
    FZ_CUDA(cudaStreamSynchronize(st));
    return h.err != 0 ? err_status(h.err) : FZ_OK;
}

fz_status fz_last_header(void* h_hdr)
{
    if (h_hdr == nullptr || !g_have_hdr) return FZ_ERR_ARG;
    memcpy(h_hdr, g_last_hdr, 128);
    return FZ_OK;
}

fz_status fz_debug_decode_q(const void* d_in, size_t in_size, int32_t* d_q, uint64_t n, void* d_work,
                            size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    if (d_q == nullptr || !aligned16(d_q)) return FZ_ERR_ARG;
    return decompress_impl(d_in, in_size, nullptr, d_q, n, d_work, work_bytes,
                           static_cast<cudaStream_t>(stream));
}

fz_status fz_compress_host(const float* h_field, const fz_shape* s, int eb_mode, double eb, void* h_out,
                           size_t out_cap, size_t* out_size, float* d_field_scratch, void* d_out_scratch,
                           size_t d_out_cap, void* d_work, size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    uint64_t n;
    if (!shape_n(s, &n) || h_field == nullptr || h_out == nullptr || out_size == nullptr)
        return FZ_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FZ_CUDA(cudaMemcpyAsync(d_field_scratch, h_field, 4 * n, cudaMemcpyHostToDevice, st));
    fz_status rs = compress_impl(d_field_scratch, s, nullptr, eb_mode, eb, d_out_scratch, d_out_cap,
                                 out_size, d_work, work_bytes, st);
    if (rs != FZ_OK) return rs;
    if (*out_size > out_cap) return FZ_ERR_CAPACITY;
    FZ_CUDA(cudaMemcpyAsync(h_out, d_out_scratch, *out_size, cudaMemcpyDeviceToHost, st));
    FZ_CUDA(cudaStreamSynchronize(st));
    return FZ_OK;
}

fz_status fz_decompress_host(const void* h_in, size_t in_size, float* h_field, uint64_t n,
                             void* d_in_scratch, float* d_field_scratch, void* d_work, size_t work_bytes,
                             void* stream)
{
    LaunchScope ls(__func__);
    if (h_in == nullptr || h_field == nullptr) return FZ_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FZ_CUDA(cudaMemcpyAsync(d_in_scratch, h_in, in_size, cudaMemcpyHostToDevice, st));
    fz_status rs = decompress_impl(d_in_scratch, in_size, d_field_scratch, nullptr, n, d_work,
                                   work_bytes, st);
    if (rs != FZ_OK) return rs;
    FZ_CUDA(cudaMemcpyAsync(h_field, d_field_scratch, 4 * n, cudaMemcpyDeviceToHost, st));
    FZ_CUDA(cudaStreamSynchronize(st));
    return FZ_OK;
}

const char* fz_strerror(int status)
{
    switch (status) {
        case FZ_OK: return "ok";
        case FZ_ERR_ARG: return "invalid argument";
        case FZ_ERR_NONFINITE: return "non-finite value in the field";
        case FZ_ERR_EB_TOO_SMALL: return "error bound too small for fp32";
        case FZ_ERR_CAPACITY: return "output buffer too small";
        case FZ_ERR_CORRUPT: return "corrupt stream";
        case FZ_ERR_WORKSPACE: return "workspace too small";
        case FZ_ERR_CUDA: return "CUDA error";
        default: return "unknown status";
    }
}

const char* fz_last_cuda_error(void) { return g_cuda_err; }

void fz_debug_set_variant(int bits) { fz::set_variant_bits(bits); }

int fz_last_launch_count(void) { return g_last_launches; }

void fz_profile_enable(int on)
{
    std::lock_guard<std::mutex> g(fz::g_prof_mu);
    fz::g_prof_on = on != 0;
    fz::g_prof_mask = ~0ull;
}

void fz_profile_mask(unsigned long long mask)
{
    std::lock_guard<std::mutex> g(fz::g_prof_mu);
    fz::g_prof_mask = mask;
}

int fz_profile_timeline(int* h_ids, float* h_start_ms, float* h_end_ms, int max_records)
{
    std::lock_guard<std::mutex> g(fz::g_prof_mu);
    const int n = (int)fz::g_prof_pending.size() < max_records ? (int)fz::g_prof_pending.size() : max_records;
    if (n == 0) return 0;
    const cudaEvent_t t0 = fz::g_prof_pending[0]->a;
    for (int k = 0; k < n; ++k) {
        const fz::ProfRec& r = *fz::g_prof_pending[k];
        if (r.done) cudaEventSynchronize(r.b);
        float a = 0.0f, b = 0.0f;
        cudaEventElapsedTime(&a, t0, r.a);
        if (r.done) cudaEventElapsedTime(&b, t0, r.b);
        if (h_ids) h_ids[k] = r.id;
        if (h_start_ms) h_start_ms[k] = a;
        if (h_end_ms) h_end_ms[k] = b;
    }
    return n;
}

int fz_profile_read(double* h_ms, int* h_launches, int max_kernels)
{
    std::lock_guard<std::mutex> g(fz::g_prof_mu);
    size_t keep = 0;
    for (fz::ProfRec* r : fz::g_prof_pending) {
        if (!r->done) {                       // launch still being issued by another thread
            fz::g_prof_pending[keep++] = r;
            continue;
        }
        cudaEventSynchronize(r->b);
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, r->a, r->b) == cudaSuccess) {
            fz::g_prof_ms[r->id] += ms;
            fz::g_prof_n[r->id] += 1;
        }
        fz::g_prof_pool.push_back(r->a);
        fz::g_prof_pool.push_back(r->b);
        delete r;
    }
    fz::g_prof_pending.resize(keep);
    for (int k = 0; k < fz::K_COUNT && k < max_kernels; ++k) {
        if (h_ms) h_ms[k] = fz::g_prof_ms[k];
        if (h_launches) h_launches[k] = fz::g_prof_n[k];
        fz::g_prof_ms[k] = 0.0;
        fz::g_prof_n[k] = 0;
    }
    return fz::K_COUNT;
}

const char* fz_kernel_name(int id)
{
    static const char* names[] = {"k_init", "k_range", "k_params", "k_compress", "k_finalize",
                                  "k_decode_init", "k_validate_outliers", "k_decode_tiles",
                                  "k_scan_sums", "k_scan_chunks", "k_scan_apply", "k_value_patch",
                                  "k_outliers", "k_tile_offsets", "k_xcarry", "k_slab", "k_decode_planes",
                                  "k_scan_walk", "k_compact", "k_dzr_sum", "k_dzr_prep", "k_dzr_main", "k_logt", "k_rowtiles"};
    return (id >= 0 && id < fz::K_COUNT) ? names[id] : "?";
}

// ---------------------------------------------------------------------------------------
// Slab API (multi-GPU z-slabs, SV §8.e)
// ---------------------------------------------------------------------------------------
fz_status fz_slab_range(const float* d_slab, uint64_t n, float* h_min, float* h_max, int64_t* h_first_bad,
                        void* d_work, size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    if (d_slab == nullptr || !aligned16(d_slab) || d_work == nullptr || work_bytes < 512 || n == 0)
        return FZ_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Ctrl* ctrl = static_cast<Ctrl*>(d_work);
    FZ_CUDA(launch_init(ctrl, nullptr, nullptr, 0, nullptr, st));
    FZ_CUDA(launch_range(d_slab, n, ctrl, st));
    Ctrl h;
    FZ_CUDA(cudaMemcpyAsync(&h, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    FZ_CUDA(cudaStreamSynchronize(st));
    if (h_min) *h_min = ord2f(h.mn_enc);
    if (h_max) *h_max = ord2f(h.mx_enc);
    if (h_first_bad) *h_first_bad = h.first_bad == ~0ull ? -1 : (int64_t)h.first_bad;
    return h.first_bad == ~0ull ? FZ_OK : FZ_ERR_NONFINITE;
}

size_t fz_slab_stage_bound(const fz_shape* global, uint64_t tb, uint64_t te)
{
    uint64_t n;
    if (!shape_n(global, &n) || te <= tb || te > tiles_of(n)) return 0;
    const uint64_t nt = te - tb;
    const uint64_t e1 = te * kTileCodes < n ? te * kTileCodes : n;
    const uint64_t elems = e1 - tb * kTileCodes;
    return (size_t)(32 * nt + 4096 * nt + 16 * elems);
}

fz_status fz_slab_compress(const float* d_slab, uint64_t slab_first, uint64_t slab_elems,
                           const fz_shape* global, uint64_t tb, uint64_t te, const fz_params* p,
                           void* d_stage, size_t stage_cap, fz_counts* h_counts, void* d_work,
                           size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    uint64_t n;
    if (!shape_n(global, &n) || d_slab == nullptr || p == nullptr || d_stage == nullptr ||
        h_counts == nullptr || d_work == nullptr || !aligned16(d_slab) || !aligned16(d_stage) ||
        !aligned16(d_work) || (slab_first & 3) != 0 || (p->mode & ~FZ_CHUNK_LOCAL) == FZ_EB_PWREL)
        return FZ_ERR_ARG;   // (f3's log transform is not part of the slab protocol)
    const uint64_t T = tiles_of(n);
    if (te <= tb || te > T) return FZ_ERR_ARG;
    const Geom g = geom_of(*global, n);
    const uint64_t halo = (uint64_t)(global->ndim == 3 ? g.P : 0) + (global->ndim >= 2 ? g.nx : 0) + 1;
    const uint64_t need_lo = tb * kTileCodes > halo ? tb * kTileCodes - halo : 0;
    const uint64_t need_hi = te * kTileCodes < n ? te * kTileCodes : n;
    if (slab_first > need_lo || slab_first + slab_elems < need_hi) return FZ_ERR_ARG;
    Work W{layout_of(*global, n, T), static_cast<uint8_t*>(d_work)};
    if (work_bytes < W.L.total) return FZ_ERR_WORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t nt = te - tb;
    uint8_t* stage = static_cast<uint8_t*>(d_stage);
    const bool cl = (p->mode & FZ_CHUNK_LOCAL) != 0;
    if (cl && !cl_slab(*global, n, tb, te)) return FZ_ERR_ARG;
    fz_params pm = *p;
    pm.mode &= ~FZ_CHUNK_LOCAL;
    p = &pm;

    CompressArgs a = make_args(W, d_slab, slab_first, g, (uint32_t)tb, (uint32_t)te);
    a.cl = cl ? 1u : 0u;
    a.flags_out = stage;
    a.flags_cap = stage_cap < 32 * nt ? stage_cap : 32 * nt;
    a.payload_out = stage + 32 * nt;
    a.payload_cap = stage_cap > 32 * nt ? stage_cap - 32 * nt : 0;
    Ctrl h;
    fz_status rs = compress_run(W, a, p, (int)p->mode, p->eb_input, nullptr, 0, *global, n, &h, st);
    if (rs != FZ_OK) return rs;
    if (h.err != 0) return err_status(h.err);
    h_counts->nnz = h.nnz;
    h_counts->n_delta = h.nd;
    h_counts->n_value = h.nv;
    const uint64_t dbase = 32 * nt + 16 * h.nnz, vbase = dbase + 8 * h.nd, need = vbase + 8 * h.nv;
    if (need > stage_cap) return FZ_ERR_CAPACITY;
    OutDest d;
    d.drec = reinterpret_cast<uint2*>(stage + dbase);
    d.vrec = reinterpret_cast<uint2*>(stage + vbase);
    return place_outliers(W, a, h, d, st);
}

fz_status fz_slab_place(const void* d_stage, const fz_shape* global, uint64_t tb, uint64_t te,
                        const fz_counts* local, const fz_counts* before, const fz_counts* totals,
                        const fz_params* p, int write_header, void* d_out, size_t out_cap, void* stream)
{
    LaunchScope ls(__func__);
    uint64_t n;
    if (!shape_n(global, &n) || d_stage == nullptr || local == nullptr || before == nullptr ||
        totals == nullptr || d_out == nullptr || (write_header && p == nullptr))
        return FZ_ERR_ARG;
    const uint64_t T = tiles_of(n);
    if (te <= tb || te > T) return FZ_ERR_ARG;
    const uint64_t nt = te - tb;
    const uint64_t total = kHeaderBytes + 32 * T + 16 * totals->nnz + 8 * totals->n_delta + 8 * totals->n_value;
    if (total > out_cap) return FZ_ERR_CAPACITY;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint8_t* s8 = static_cast<const uint8_t*>(d_stage);
    uint8_t* o = static_cast<uint8_t*>(d_out);
    const uint64_t pbase = kHeaderBytes + 32 * T, dbase = pbase + 16 * totals->nnz,
                   vbase = dbase + 8 * totals->n_delta;
    const uint64_t sd = 32 * nt + 16 * local->nnz, sv = sd + 8 * local->n_delta;
    FZ_CUDA(cudaMemcpyAsync(o + kHeaderBytes + 32 * tb, s8, 32 * nt, cudaMemcpyDeviceToDevice, st));
    if (local->nnz)
        FZ_CUDA(cudaMemcpyAsync(o + pbase + 16 * before->nnz, s8 + 32 * nt, 16 * local->nnz, cudaMemcpyDeviceToDevice, st));
    if (local->n_delta)
        FZ_CUDA(cudaMemcpyAsync(o + dbase + 8 * before->n_delta, s8 + sd, 8 * local->n_delta, cudaMemcpyDeviceToDevice, st));
    if (local->n_value)
        FZ_CUDA(cudaMemcpyAsync(o + vbase + 8 * before->n_value, s8 + sv, 8 * local->n_value, cudaMemcpyDeviceToDevice, st));
    if (write_header) {
        uint8_t h[128];
        const bool cl = (p->mode & FZ_CHUNK_LOCAL) != 0;
        fz_params pm = *p;
        pm.mode &= ~FZ_CHUNK_LOCAL;
        write_header_host(h, *global, n, T, pm, *totals, total, cl ? cl_chunk(*global) : 0u);
        FZ_CUDA(cudaMemcpyAsync(o, h, 128, cudaMemcpyHostToDevice, st));
    }
    FZ_CUDA(cudaStreamSynchronize(st));
    return FZ_OK;
}

fz_status fz_debug_quantize(const float* d_field, const fz_shape* s, const fz_params* p, uint16_t* d_codes,
                            uint32_t* d_didx, int32_t* d_dval, uint64_t dcap, uint64_t* h_nd,
                            uint32_t* d_vidx, uint32_t* d_vbits, uint64_t vcap, uint64_t* h_nv,
                            void* d_work, size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    uint64_t n;
    if (!shape_n(s, &n) || d_field == nullptr || p == nullptr || d_codes == nullptr || h_nd == nullptr ||
        h_nv == nullptr || !aligned16(d_field) || !aligned16(d_work))
        return FZ_ERR_ARG;
    const uint64_t T = tiles_of(n);
    Work W{layout_of(*s, n, T), static_cast<uint8_t*>(d_work)};
    // the hook runs the product kernels, which write flags and payload: scratch for them
    // follows the compression workspace (fz_debug_workspace_bytes)
    if (work_bytes < W.L.total + 32 * T + 4096 * T) return FZ_ERR_WORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CompressArgs a = make_args(W, d_field, 0, geom_of(*s, n), 0, (uint32_t)T);
    a.codes_out = d_codes;
    a.flags_out = static_cast<uint8_t*>(d_work) + W.L.total;
    a.flags_cap = 32 * T;
    a.payload_out = a.flags_out + 32 * T;
    a.payload_cap = 4096 * T;
    Ctrl h;
    fz_status rs = compress_run(W, a, p, (int)p->mode, p->eb_input, nullptr, 0, *s, n, &h, st);
    if (rs != FZ_OK) return rs;
    if (h.err != 0) return err_status(h.err);
    *h_nd = h.nd;
    *h_nv = h.nv;
    if (h.nd > dcap || h.nv > vcap) return FZ_ERR_CAPACITY;
    OutDest d;
    d.didx = d_didx;
    d.dval = d_dval;
    d.vidx = d_vidx;
    d.vbits = d_vbits;
    return place_outliers(W, a, h, d, st);
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// Slab decompression (multi-GPU, plane-aligned z-slabs)
// ---------------------------------------------------------------------------------------
namespace {
struct SlabGeo {
    fz_shape local;     // the slab as a standalone field
    uint64_t n, g0;     // local elements, global index of local element 0
    uint64_t L, W;      // slowest-axis length and the aggregate width
};

fz_status slab_geo(const fz_shape* global, uint64_t tb, uint64_t te, SlabGeo* sg)
{
    uint64_t n;
    if (!shape_n(global, &n)) return FZ_ERR_ARG;
    const uint64_t T = tiles_of(n);
    if (te <= tb || te > T) return FZ_ERR_ARG;
    const uint64_t g0 = tb * kTileCodes, g1 = te * kTileCodes < n ? te * kTileCodes : n;
    const Geom g = geom_of(*global, n);
    const uint64_t unit = global->ndim == 3 ? g.P : (global->ndim == 2 ? g.nx : 1);
    if (g0 % unit != 0 || (g1 != n && g1 % unit != 0)) return FZ_ERR_ARG;   // not plane-aligned
    SlabGeo r{};
    r.n = g1 - g0;
    r.g0 = g0;
    r.local = *global;
    r.local.dims[0] = r.n / unit;
    r.L = r.local.dims[0];
    r.W = unit;
    *sg = r;
    return FZ_OK;
}
}  // namespace

extern "C" {

uint64_t fz_slab_agg_elems(const fz_shape* global)
{
    uint64_t n;
    if (!shape_n(global, &n)) return 0;
    const Geom g = geom_of(*global, n);
    return global->ndim == 3 ? g.P : (global->ndim == 2 ? g.nx : 1);
}

fz_status fz_slab_decode(const void* d_stage, const fz_counts* local, const fz_shape* global, uint64_t tb,
                         uint64_t te, int32_t* d_q, int32_t* d_agg, void* d_work, size_t work_bytes, void* stream)
{
    LaunchScope ls(__func__);
    SlabGeo sg;
    if (d_stage == nullptr || local == nullptr || d_q == nullptr || d_agg == nullptr || d_work == nullptr ||
        !aligned16(d_stage) || !aligned16(d_q) || !aligned16(d_work))
        return FZ_ERR_ARG;
    fz_status rs = slab_geo(global, tb, te, &sg);
    if (rs != FZ_OK) return rs;
    const DecodeLayout L = decode_layout(sg.local);
    if (work_bytes < L.total) return FZ_ERR_WORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* wb = static_cast<uint8_t*>(d_work);
    Ctrl* ctrl = reinterpret_cast<Ctrl*>(wb + L.ctrl);
    const uint64_t nt = te - tb;
    const uint8_t* in = static_cast<const uint8_t*>(d_stage);
    const uint64_t pbase = 32 * nt, dbase = pbase + 16 * local->nnz;
    const Geom g = geom_of(sg.local, sg.n);
    FZ_CUDA(launch_decode_init(ctrl, st));
    FZ_CUDA(launch_tile_offsets(in, (uint32_t)nt, reinterpret_cast<uint32_t*>(wb + L.loc),
                                reinterpret_cast<uint32_t*>(wb + L.bsum), ctrl, st, local->nnz));
    FZ_CUDA(launch_record_tiles(reinterpret_cast<const uint2*>(in + dbase), local->n_delta, (uint32_t)nt, sg.g0,
                                reinterpret_cast<uint32_t*>(wb + L.drange), st));
    DecodeArgs a{};
    a.flags = in;
    a.payload = in + pbase;
    a.drec = reinterpret_cast<const uint2*>(in + dbase);
    a.drange = reinterpret_cast<const uint32_t*>(wb + L.drange);
    a.nnz_total = local->nnz;
    a.nd = local->n_delta;
    a.g = g;
    a.tiles = (uint32_t)nt;
    a.w = 0.0f;
    a.q_out = d_q;
    a.gbase = sg.g0;
    a.loc = reinterpret_cast<const uint32_t*>(wb + L.loc);
    a.bpre = reinterpret_cast<const uint32_t*>(wb + L.bsum);
    a.xagg = reinterpret_cast<uint2*>(wb + L.xagg);
    a.ctrl = ctrl;
    FZ_CUDA(launch_decode_tiles(a, st));
    const bool carries = nt > 1 && (g.ndim == 1 || !(g.nx <= kTileCodes && kTileCodes % g.nx == 0));
    if (carries)
        FZ_CUDA(launch_xcarry(a, reinterpret_cast<uint2*>(wb + L.xloc), reinterpret_cast<uint2*>(wb + L.xbagg), true, st));
    if (sg.local.ndim == 3)
        FZ_CUDA(launch_scan_axis(d_q, sg.local.dims[0], sg.local.dims[1], sg.local.dims[2],
                                 reinterpret_cast<uint32_t*>(wb + L.sums), 0.0f, st));
    if (sg.local.ndim >= 2) FZ_CUDA(launch_axis_sum(d_q, sg.L, sg.W, d_agg, st));
    else FZ_CUDA(cudaMemcpyAsync(d_agg, d_q + (sg.n - 1), 4, cudaMemcpyDeviceToDevice, st));
    Ctrl h;
    FZ_CUDA(cudaMemcpyAsync(&h, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    FZ_CUDA(cudaStreamSynchronize(st));
    if (h.err != 0) return err_status(h.err);
    if (h.nnz != local->nnz) return FZ_ERR_CORRUPT;
    return FZ_OK;
}

fz_status fz_slab_decode_cl(const void* d_stage, const fz_counts* local, const fz_shape* global, uint64_t tb,
                            uint64_t te, const fz_params* p, float* d_out, void* d_work, size_t work_bytes,
                            void* stream)
{
    LaunchScope ls(__func__);
    SlabGeo sg;
    uint64_t n;
    if (d_stage == nullptr || local == nullptr || p == nullptr || d_out == nullptr || d_work == nullptr ||
        !aligned16(d_stage) || !aligned16(d_out) || !aligned16(d_work) || !shape_n(global, &n))
        return FZ_ERR_ARG;
    if (!cl_slab(*global, n, tb, te)) return FZ_ERR_ARG;
    fz_status rs = slab_geo(global, tb, te, &sg);
    if (rs != FZ_OK) return rs;
    const DecodeLayout L = decode_layout(sg.local);
    if (work_bytes < L.total) return FZ_ERR_WORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* wb = static_cast<uint8_t*>(d_work);
    Ctrl* ctrl = reinterpret_cast<Ctrl*>(wb + L.ctrl);
    const uint64_t nt = te - tb;
    const uint8_t* in = static_cast<const uint8_t*>(d_stage);
    const uint64_t pbase = 32 * nt, dbase = pbase + 16 * local->nnz, vbase = dbase + 8 * local->n_delta;
    FZ_CUDA(launch_decode_init(ctrl, st));
    FZ_CUDA(launch_tile_offsets(in, (uint32_t)nt, reinterpret_cast<uint32_t*>(wb + L.loc),
                                reinterpret_cast<uint32_t*>(wb + L.bsum), ctrl, st, local->nnz));
    FZ_CUDA(launch_record_tiles(reinterpret_cast<const uint2*>(in + dbase), local->n_delta, (uint32_t)nt, sg.g0,
                                reinterpret_cast<uint32_t*>(wb + L.drange), st));
    DecodeArgs a{};
    a.flags = in;
    a.payload = in + pbase;
    a.drec = reinterpret_cast<const uint2*>(in + dbase);
    a.drange = reinterpret_cast<const uint32_t*>(wb + L.drange);
    a.nnz_total = local->nnz;
    a.nd = local->n_delta;
    a.g = geom_of(sg.local, sg.n);
    a.tiles = (uint32_t)nt;
    a.w = p->w;
    a.q_out = reinterpret_cast<int32_t*>(d_out);
    a.gbase = sg.g0;
    a.loc = reinterpret_cast<const uint32_t*>(wb + L.loc);
    a.bpre = reinterpret_cast<const uint32_t*>(wb + L.bsum);
    a.ctrl = ctrl;
    // the slab starts on a chunk boundary, so its local chunks are the global ones
    FZ_CUDA(launch_decode_cl(a, kClDepth, st));
    FZ_CUDA(launch_value_patch(d_out, reinterpret_cast<const uint2*>(in + vbase), local->n_value, sg.n, st, sg.g0));
    Ctrl h;
    FZ_CUDA(cudaMemcpyAsync(&h, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    FZ_CUDA(cudaStreamSynchronize(st));
    if (h.err != 0) return err_status(h.err);
    if (h.nnz != local->nnz) return FZ_ERR_CORRUPT;
    return FZ_OK;
}

fz_status fz_slab_carry(const int32_t* d_aggs, uint32_t nbefore, uint64_t elems, int32_t* d_carry, void* stream)
{
    LaunchScope ls(__func__);
    if (d_carry == nullptr || (nbefore > 0 && d_aggs == nullptr) || elems == 0) return FZ_ERR_ARG;
    FZ_CUDA(launch_slab_carry(d_aggs, nbefore, elems, d_carry, static_cast<cudaStream_t>(stream)));
    return FZ_OK;
}

fz_status fz_slab_finish(int32_t* d_q, const int32_t* d_carry, const void* d_stage, const fz_counts* local,
                         const fz_shape* global, uint64_t tb, uint64_t te, const fz_params* p, void* stream)
{
    LaunchScope ls(__func__);
    SlabGeo sg;
    if (d_q == nullptr || d_carry == nullptr || d_stage == nullptr || local == nullptr || p == nullptr)
        return FZ_ERR_ARG;
    fz_status rs = slab_geo(global, tb, te, &sg);
    if (rs != FZ_OK) return rs;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (sg.local.ndim >= 2) FZ_CUDA(launch_walk_carry(d_q, sg.L, sg.W, p->w, d_carry, st));
    else FZ_CUDA(launch_add_dequant(d_q, sg.n, d_carry, p->w, st));
    const uint64_t nt = te - tb;
    const uint8_t* in = static_cast<const uint8_t*>(d_stage);
    const uint2* vrec = reinterpret_cast<const uint2*>(in + 32 * nt + 16 * local->nnz + 8 * local->n_delta);
    FZ_CUDA(launch_value_patch(reinterpret_cast<float*>(d_q), vrec, local->n_value, sg.n, st, sg.g0));
    FZ_CUDA(cudaStreamSynchronize(st));
    return FZ_OK;
}

}  // extern "C"
