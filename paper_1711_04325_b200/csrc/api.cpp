// C ABI of lmsgd (include/lmsgd.h): argument checking, the per-rank context
// (exchange buffers, CUDA-IPC peer mappings, status words) and the stream-ordered
// composition of the sm_100a kernels in kernels.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "lmsgd.h"
#include "lmsgd_internal.h"

#include <nvtx3/nvToolsExt.h>   // header-only; ranges are no-ops unless a profiler is attached

using lmsgd::Layout;
using lmsgd::UpdConst;

struct lmsgd_ctx {
    int world = 1, rank = 0, device = 0;
    int64_t n = 0, n_pad = 0;
    float scale = 1.0f;
    lmsgd_hyper hyper{};
    double wd = 0.0;                  // lmsgd_set_weight_decay (R12)
    int64_t n_wd = 0;
    int64_t ctab_n_wd = 0;   // n_wd the uploaded table was built with (selects the kernel variant)
    uint32_t flags = 0;
    Layout lay{};
    char* buf = nullptr;           // own exchange buffer (IPC-shared when world > 1)
    lmsgd::Peers peers{};
    bool connected = false;
    bool group = false;               // lmsgd_connect_group: peers are in-process buffers (no IPC)
    lmsgd::XStep* d_group = nullptr;  // device XStep[LMSGD_MAX_WORLD] of a group call led by this ctx
    lmsgd::XStep* d_group_graph = nullptr;   // the same for graph mode (constant across replays)
    std::vector<lmsgd::XStep> group_graph_cache;
    lmsgd::BnArgs* d_group_bn = nullptr;
    unsigned int* tickets = nullptr;  // device [4]
    unsigned int* xctr = nullptr;     // device [4 + nchunks] counters of the world > 1 kernels
    // device-resident step state (so a captured step replays as the next step)
    struct DevState { uint32_t xepoch, bnepoch, k1epoch, pad; int64_t cursor; };
    DevState* dstate = nullptr;       // device
    lmsgd::UpdConst* d_ctab = nullptr;   // lmsgd_schedule_upload table
    int64_t ctab_count = 0, ctab_cap = 0;
    int mode = 0;                     // 0 unused, 1 lmsgd_step, 2 lmsgd_step_graph (not mixed)
    int64_t* last = nullptr;          // device lmsgd_step_status of the last step
    // lmsgd_step_host: two device staging buffers filled by a copy stream, so the
    // host->device copy of step i+1 overlaps the kernels of step i (lazy)
    float* d_grads[2] = {nullptr, nullptr};
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
    int host_buf = 0;
    uint32_t step = 0, bn_calls = 0;
    cudaStream_t last_stream = nullptr;
    lmsgd::Launch L{};
    int xblocks = 0;                  // lmsgd_set_exchange_blocks (0 = L.grid_xstep)
    int64_t timeout_ns = 10'000'000'000LL;
    std::string err;
    // profiling (lmsgd_profile_enable): event pairs around each kernel launch
    struct Rec { int phase; cudaEvent_t a, b; };
    std::vector<cudaEvent_t> pool;
    std::vector<Rec> recs;
    size_t prof_cap = 0;
    // tracing (lmsgd_trace_enable): TR_WORDS stamps per step, ring of trace_cap steps
    int64_t* d_trace = nullptr;
    int64_t trace_cap = 0, trace_steps = 0;
    // NVLS (lmsgd_nvls_*): multicast object, this rank's physical wire bound to it, and
    // its unicast and multicast mappings
    struct Nvls {
        int stage = 0;                 // 0 none, 1 created/imported + device added, 2 bound + mapped
        int mode = 0;
        bool bound = false, uc_mapped = false, mc_mapped = false;
        CUmemGenericAllocationHandle mc = 0, phys = 0;
        CUdeviceptr uc_va = 0, mc_va = 0;
        size_t size = 0;
        std::thread server;            // rank 0: hands the multicast fd to the other ranks
        int fd = -1;
    } nv;
};

namespace {

thread_local std::string g_err;  // for context-free calls

// NVTX range around a host entry point (nsys / Nsight timelines: which library call
// enqueued which kernels).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

lmsgd_status fail(lmsgd_ctx* c, lmsgd_status s, const std::string& msg) {
    if (c) c->err = msg; else g_err = msg;
    return s;
}

lmsgd_status cuda_fail(lmsgd_ctx* c, cudaError_t e, const char* what) {
    return fail(c, LMSGD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(ctx, call)                                                   \
    do {                                                                \
        cudaError_t e_ = (call);                                        \
        if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #call);      \
    } while (0)

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

bool aligned16(const void* p) { return p && (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool pow2_scale(float s) {
    if (!(s > 0.0f) || !std::isfinite(s)) return false;
    int e;
    return std::frexp(static_cast<double>(s), &e) == 0.5;
}

// Launch geometry of the current device: SMs x resident blocks of the streaming kernels.
lmsgd::Launch launch_for_current_device() {
    static lmsgd::Launch cache[64];
    static bool have[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && have[dev]) return cache[dev];
    lmsgd::Launch L{};
    cudaDeviceGetAttribute(&L.sm_count, cudaDevAttrMultiProcessorCount, dev);
    L.grid_cap_stream = L.sm_count * lmsgd::stream_blocks_per_sm();
    {
        const int occ = lmsgd::xstep_blocks_per_sm(), bps = lmsgd::xstep_default_bps();
        L.grid_xstep = L.sm_count * (bps < occ ? bps : occ);
    }
    // diagnostics: fewer k_xstep1 blocks per SM, leaving slots for k_xupdate blocks to be
    // resident early -- measured slower (k = 4: 205.0 / 207.8 us at 6 / 4 vs 203.9 us at 8,
    // profiles/r1/ab/xstep_grid_n4.txt)
    if (const char* b = std::getenv("LMSGD_XSTEP_BPS")) {
        const int bps = std::atoi(b);
        if (bps > 0 && bps <= lmsgd::xstep_blocks_per_sm()) L.grid_xstep = L.sm_count * bps;
    }
    // PDL on the k = 1 pair: 128.7 vs 132.3 us (the world > 1 step uses it internally).
    L.pdl_mask = 0x1;
    if (const char* m = std::getenv("LMSGD_PDL_MASK")) L.pdl_mask = std::atoi(m);  // diagnostics
    if (dev >= 0 && dev < 64) { cache[dev] = L; have[dev] = true; }
    return L;
}

bool coeffs_ok(const lmsgd_coeffs* c) {
    return c && std::isfinite(c->eta) && c->eta > 0.0 && c->alpha_sgd >= 0.0 && c->alpha_sgd <= 1.0 &&
           std::isfinite(c->alpha_rmsprop) && c->alpha_rmsprop >= 0.0;
}

bool hyper_ok(const lmsgd_hyper* h) {
    return h && h->mu1 >= 0.0 && h->mu1 < 1.0 && h->mu2 >= 0.0 && h->mu2 < 1.0 && h->eps > 0.0 &&
           std::isfinite(h->eps);
}

// fp32 constants rounded once from double (R15: fp32(1 - mu2), not 1 - fp32(mu2)).
UpdConst make_const(const lmsgd_hyper& h, const lmsgd_coeffs& c, int k, float s, double wd = 0.0,
                    int64_t n_wd = 0) {
    UpdConst u{};
    u.wd = static_cast<float>(wd);
    u.n_wd = wd > 0.0 ? n_wd : 0;   // wd = 0: the decay branch is never taken (keeps -0.0 exact)
    u.mu1 = static_cast<float>(h.mu1);
    u.mu2 = static_cast<float>(h.mu2);
    u.omm2 = static_cast<float>(1.0 - h.mu2);
    u.eps = static_cast<float>(h.eps);
    u.eta = static_cast<float>(c.eta);
    u.a_sgd = static_cast<float>(c.alpha_sgd);
    u.a_rms = static_cast<float>(c.alpha_rmsprop);
    u.inv_ks = static_cast<float>(1.0 / (static_cast<double>(k) * static_cast<double>(s)));
    return u;
}

Layout make_layout(int world, int64_t n) {
    Layout L{};
    L.shard = align_up((n + world - 1) / world, 64);
    if (L.shard == 0) L.shard = 64;
    L.off_recv = 0;
    int64_t off = align_up(L.off_recv + 2 * L.shard * world, 256);
    if (world > 1) {
        L.off_R = off;
        off = align_up(off + 2 * L.shard, 256);
    } else {
        L.off_R = L.off_recv;  // k = 1: the packed buffer is the all-reduce result
    }
    L.off_status = off;
    off = align_up(off + 2 * lmsgd::ST_WORDS * 8, 256);
    L.off_flags = off;
    off = align_up(off + 4 * 128, 256);
    L.off_bn = off;
    if (world > 1) off = align_up(off + int64_t(2) * 2 * LMSGD_MAX_BN_CHANNELS * 4, 256);
    // reduce chunks: 32 units of 2048 elements (64K elements) of the shard each
    const int64_t units_per_shard = (L.shard / 8 + 255) / 256;
    L.cu = 32;
    L.nchunks = static_cast<int32_t>((units_per_shard + L.cu - 1) / L.cu);
    L.off_cflags = off;
    if (world > 1) off = align_up(off + int64_t(L.nchunks) * LMSGD_MAX_WORLD * 4, 256);
    L.bytes = off;
    return L;
}

int64_t* status_slot(lmsgd_ctx* c, int parity) {
    return reinterpret_cast<int64_t*>(c->buf + c->lay.off_status) + parity * lmsgd::ST_WORDS;
}

lmsgd::XArgs xargs(lmsgd_ctx* c, uint32_t epoch, uint32_t* dev_epoch) {
    lmsgd::XArgs x{};
    x.peers = c->peers;
    x.lay = c->lay;
    x.world = c->world;
    x.rank = c->rank;
    x.epoch = epoch;
    x.parity = static_cast<int>(epoch & 1u);
    x.n = c->n;
    x.timeout_ns = c->timeout_ns;
    x.ticket = c->tickets;
    x.dev_epoch = dev_epoch;
    x.trace = nullptr;
    x.nv = c->nv.stage == 2 ? c->nv.mode : 0;
    x.nv_uc = reinterpret_cast<char*>(c->nv.uc_va);
    x.nv_mc = reinterpret_cast<char*>(c->nv.mc_va);
    if (c->d_trace) {
        x.trace = c->d_trace + (c->trace_steps % c->trace_cap) * lmsgd::TR_WORDS;
        ++c->trace_steps;
    }
    return x;
}

// Device-guard: make ctx->device current for the duration of a call.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Launch one kernel, bracketed by profiling events when enabled.
template <class F>
cudaError_t timed(lmsgd_ctx* c, cudaStream_t s, int phase, F&& launch) {
    const bool rec = c->prof_cap > 0 && c->recs.size() < c->prof_cap && c->pool.size() >= 2;
    lmsgd_ctx::Rec r{phase, nullptr, nullptr};
    if (rec) {
        r.b = c->pool.back(); c->pool.pop_back();
        r.a = c->pool.back(); c->pool.pop_back();
        cudaEventRecord(r.a, s);
    }
    cudaError_t e = launch();
    if (rec) {
        cudaEventRecord(r.b, s);
        c->recs.push_back(r);
    }
    return e;
}


// ---------------------------------------------------------------- NVLS plumbing
// Driver API entry points (through the runtime: no link-time dependency on libcuda).
struct Drv {
    PFN_cuGetErrorString_v6000 errStr = nullptr;
    PFN_cuDeviceGet_v2000 devGet = nullptr;
    PFN_cuDeviceGetAttribute_v2000 devAttr = nullptr;
    PFN_cuMulticastCreate_v12010 mcCreate = nullptr;
    PFN_cuMulticastAddDevice_v12010 mcAdd = nullptr;
    PFN_cuMulticastBindMem_v12010 mcBind = nullptr;
    PFN_cuMulticastUnbind_v12010 mcUnbind = nullptr;
    PFN_cuMulticastGetGranularity_v12010 mcGran = nullptr;
    PFN_cuMemCreate_v10020 memCreate = nullptr;
    PFN_cuMemRelease_v10020 memRelease = nullptr;
    PFN_cuMemMap_v10020 memMap = nullptr;
    PFN_cuMemUnmap_v10020 memUnmap = nullptr;
    PFN_cuMemAddressReserve_v10020 addrReserve = nullptr;
    PFN_cuMemAddressFree_v10020 addrFree = nullptr;
    PFN_cuMemSetAccess_v10020 setAccess = nullptr;
    PFN_cuMemGetAllocationGranularity_v10020 memGran = nullptr;
    PFN_cuMemExportToShareableHandle_v10020 exportH = nullptr;
    PFN_cuMemImportFromShareableHandle_v10020 importH = nullptr;
    bool ok = false;
};

Drv load_drv() {
    Drv d;
    bool ok = true;
    auto get = [&](const char* name, auto& fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) ok = false;
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
    };
    get("cuGetErrorString", d.errStr);
    get("cuDeviceGet", d.devGet);
    get("cuDeviceGetAttribute", d.devAttr);
    get("cuMulticastCreate", d.mcCreate);
    get("cuMulticastAddDevice", d.mcAdd);
    get("cuMulticastBindMem", d.mcBind);
    get("cuMulticastUnbind", d.mcUnbind);
    get("cuMulticastGetGranularity", d.mcGran);
    get("cuMemCreate", d.memCreate);
    get("cuMemRelease", d.memRelease);
    get("cuMemMap", d.memMap);
    get("cuMemUnmap", d.memUnmap);
    get("cuMemAddressReserve", d.addrReserve);
    get("cuMemAddressFree", d.addrFree);
    get("cuMemSetAccess", d.setAccess);
    get("cuMemGetAllocationGranularity", d.memGran);
    get("cuMemExportToShareableHandle", d.exportH);
    get("cuMemImportFromShareableHandle", d.importH);
    d.ok = ok;
    return d;
}

const Drv& drv() {
    static const Drv d = load_drv();   // thread-safe one-time initialisation
    return d;
}

lmsgd_status drv_fail(lmsgd_ctx* c, CUresult r, const char* what) {
    const char* m = nullptr;
    if (drv().errStr) drv().errStr(r, &m);
    return fail(c, LMSGD_ERR_CUDA, std::string(what) + ": " + (m ? m : "driver error " + std::to_string(r)));
}

#define CKD(ctx, call)                                                  \
    do {                                                                \
        CUresult r_ = (call);                                           \
        if (r_ != CUDA_SUCCESS) return drv_fail((ctx), r_, #call);      \
    } while (0)

// The NVLS handle (LMSGD_NVLS_HANDLE_BYTES): where to fetch the multicast fd, and the size.
struct NvHandle {
    uint32_t magic;        // 'LMNV'
    uint32_t world;
    uint64_t size;         // bytes of the multicast object (and of every rank's wire)
    char name[48];         // abstract unix socket of rank 0's fd server (NUL-terminated)
};
static_assert(sizeof(NvHandle) == LMSGD_NVLS_HANDLE_BYTES, "NVLS handle size");
constexpr uint32_t kNvMagic = 0x564e4d4cu;

socklen_t abstract_addr(const char* name, sockaddr_un* a) {
    std::memset(a, 0, sizeof *a);
    a->sun_family = AF_UNIX;
    const size_t len = std::strlen(name);
    std::memcpy(a->sun_path + 1, name, len);   // sun_path[0] = 0: the abstract namespace
    return static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + len);
}

// Rank 0: hand `fd` to `peers` connections (SCM_RIGHTS), then close the listening socket.
void fd_server(int lfd, int fd, int peers) {
    for (int i = 0; i < peers; ++i) {
        pollfd p{lfd, POLLIN, 0};
        if (poll(&p, 1, 60000) <= 0) break;   // a minute without a peer: give up
        const int cfd = accept(lfd, nullptr, nullptr);
        if (cfd < 0) break;
        char byte = 'f';
        iovec io{&byte, 1};
        alignas(cmsghdr) char ctl[CMSG_SPACE(sizeof(int))] = {};
        msghdr m{};
        m.msg_iov = &io;
        m.msg_iovlen = 1;
        m.msg_control = ctl;
        m.msg_controllen = sizeof ctl;
        cmsghdr* cm = CMSG_FIRSTHDR(&m);
        cm->cmsg_level = SOL_SOCKET;
        cm->cmsg_type = SCM_RIGHTS;
        cm->cmsg_len = CMSG_LEN(sizeof(int));
        std::memcpy(CMSG_DATA(cm), &fd, sizeof(int));
        (void)sendmsg(cfd, &m, 0);
        close(cfd);
    }
    close(lfd);
}

// Other ranks: fetch the fd from rank 0's server (retried while it comes up).
int fd_fetch(const char* name) {
    for (int attempt = 0; attempt < 600; ++attempt) {
        const int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
        if (s < 0) return -1;
        sockaddr_un a;
        const socklen_t al = abstract_addr(name, &a);
        if (connect(s, reinterpret_cast<sockaddr*>(&a), al) == 0) {
            char byte = 0;
            iovec io{&byte, 1};
            alignas(cmsghdr) char ctl[CMSG_SPACE(sizeof(int))] = {};
            msghdr m{};
            m.msg_iov = &io;
            m.msg_iovlen = 1;
            m.msg_control = ctl;
            m.msg_controllen = sizeof ctl;
            int fd = -1;
            if (recvmsg(s, &m, 0) > 0) {
                cmsghdr* cm = CMSG_FIRSTHDR(&m);
                if (cm && cm->cmsg_type == SCM_RIGHTS) std::memcpy(&fd, CMSG_DATA(cm), sizeof(int));
            }
            close(s);
            return fd;
        }
        close(s);
        usleep(100000);
    }
    return -1;
}

void nvls_release(lmsgd_ctx* c) {
    auto& nv = c->nv;
    if (nv.server.joinable()) nv.server.join();
    if (nv.fd >= 0) { close(nv.fd); nv.fd = -1; }
    if (nv.stage == 0 || !drv().ok) return;
    const Drv& d = drv();
    if (nv.mc_va) { if (nv.mc_mapped) d.memUnmap(nv.mc_va, nv.size); d.addrFree(nv.mc_va, nv.size); }
    if (nv.uc_va) { if (nv.uc_mapped) d.memUnmap(nv.uc_va, nv.size); d.addrFree(nv.uc_va, nv.size); }
    CUdevice dev = 0;
    if (nv.bound && d.devGet(&dev, c->device) == CUDA_SUCCESS) d.mcUnbind(nv.mc, dev, 0, nv.size);
    if (nv.phys) d.memRelease(nv.phys);
    if (nv.mc) d.memRelease(nv.mc);
    nv = lmsgd_ctx::Nvls{};
}

lmsgd_status nvls_pre(lmsgd_ctx* c) {
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (c->world < 2) return fail(c, LMSGD_ERR_UNSUPPORTED, "NVLS needs world > 1");
    if (c->group) return fail(c, LMSGD_ERR_UNSUPPORTED, "NVLS needs one GPU per rank (not an emulated group)");
    if (!drv().ok) return fail(c, LMSGD_ERR_UNSUPPORTED, "driver has no multicast entry points");
    return LMSGD_OK;
}

CUmulticastObjectProp mc_prop(int world, size_t size) {
    CUmulticastObjectProp p{};
    p.numDevices = static_cast<unsigned>(world);
    p.size = size;
    p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    p.flags = 0;
    return p;
}
// The launch geometry of ctx's world > 1 kernels: k_xstep1's grid capped by
// lmsgd_set_exchange_blocks.
lmsgd::Launch xlaunch(const lmsgd_ctx* c) {
    lmsgd::Launch L = c->L;
    if (c->xblocks > 0 && c->xblocks < L.grid_xstep) L.grid_xstep = c->xblocks;
    return L;
}

}  // namespace

namespace {
lmsgd_status group_check(lmsgd_ctx* const* ctxs, int count, bool need_group) {
    if (!ctxs || count < 1 || count > LMSGD_MAX_WORLD) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "group: bad ctxs/count");
    uint32_t seen = 0;
    for (int i = 0; i < count; ++i) {
        lmsgd_ctx* c = ctxs[i];
        if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "group: NULL context");
        if (c->world < 2 || count > c->world) return fail(c, LMSGD_ERR_INVALID_ARG, "group: world must be >= 2 and >= count");
        if (c->device != ctxs[0]->device || c->world != ctxs[0]->world || c->n != ctxs[0]->n ||
            c->scale != ctxs[0]->scale)
            return fail(c, LMSGD_ERR_INVALID_ARG, "group: contexts differ in device, world, n_params or loss scale");
        if (seen & (1u << c->rank)) return fail(c, LMSGD_ERR_INVALID_ARG, "group: a rank appears twice");
        seen |= 1u << c->rank;
        if (need_group && !(c->connected && c->group))
            return fail(c, LMSGD_ERR_STATE, "group: lmsgd_connect_group has not been called");
    }
    return LMSGD_OK;
}

// An emulated group's update may use 256-bit accesses only if every rank's state is
// 32-byte aligned (one kernel instantiation serves all ranks).
void set_group_v8(std::vector<lmsgd::XStep>& v) {
    bool all = true;
    for (const auto& a : v)
        for (const void* p : {static_cast<const void*>(a.th), static_cast<const void*>(a.d), static_cast<const void*>(a.m)})
            all = all && (reinterpret_cast<uintptr_t>(p) & 31u) == 0;
    for (auto& a : v) a.v8 = all ? 1 : 0;
}

// Upload the per-rank arguments (pageable -> device, stream-ordered) into *dbuf.
template <typename T>
lmsgd_status group_upload(lmsgd_ctx* lead, cudaStream_t s, T** dbuf, const std::vector<T>& v) {
    if (!*dbuf) CK(lead, cudaMalloc(dbuf, LMSGD_MAX_WORLD * sizeof(T)));
    CK(lead, cudaMemcpyAsync(*dbuf, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return LMSGD_OK;
}
}  // namespace

extern "C" {

int lmsgd_abi_version(void) { return LMSGD_ABI_VERSION; }

const char* lmsgd_status_string(lmsgd_status s) {
    switch (s) {
        case LMSGD_OK: return "ok";
        case LMSGD_ERR_INVALID_ARG: return "invalid argument";
        case LMSGD_ERR_CUDA: return "CUDA error";
        case LMSGD_ERR_NONFINITE: return "non-finite gradient (step skipped)";
        case LMSGD_ERR_STATE: return "call out of order";
        case LMSGD_ERR_UNSUPPORTED: return "unsupported";
        case LMSGD_ERR_TIMEOUT: return "cross-GPU wait timed out (step skipped)";
        case LMSGD_ERR_RANGE: return "schedule step out of range";
    }
    return "unknown status";
}

lmsgd_status lmsgd_layout(int world, int64_t n, int64_t* shard, int64_t* n_pad) {
    if (world < 1 || world > LMSGD_MAX_WORLD || n < 1 || n > (int64_t(1) << 36) || !shard || !n_pad)
        return fail(nullptr, LMSGD_ERR_INVALID_ARG, "layout: bad world, n or NULL output");
    const Layout L = make_layout(world, n);
    *shard = L.shard;
    *n_pad = L.shard * world;
    return LMSGD_OK;
}

const char* lmsgd_last_error(const lmsgd_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

lmsgd_status lmsgd_init(lmsgd_ctx** out, int world, int rank, int device, int64_t n_params,
                        float loss_scale, const lmsgd_hyper* hyper, uint32_t flags) {
    if (!out) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (world < 1 || world > LMSGD_MAX_WORLD)
        return fail(nullptr, LMSGD_ERR_UNSUPPORTED, "world must be in [1, LMSGD_MAX_WORLD]");
    if (rank < 0 || rank >= world) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "rank out of range");
    if (n_params < 1 || n_params > (int64_t(1) << 36))
        return fail(nullptr, LMSGD_ERR_INVALID_ARG, "n_params out of range");
    if (!pow2_scale(loss_scale))
        return fail(nullptr, LMSGD_ERR_INVALID_ARG, "loss_scale must be a positive power of two");
    lmsgd_hyper h{};
    if (hyper) h = *hyper; else lmsgd_hyper_default(&h);
    if (!hyper_ok(&h)) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "hyperparameters out of range");
    if (flags & ~(LMSGD_FLAG_NO_SKIP | LMSGD_FLAG_FREEZE_M)) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "unknown flags");

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return fail(nullptr, LMSGD_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "device out of range");

    auto* c = new lmsgd_ctx();
    c->world = world; c->rank = rank; c->device = device; c->n = n_params;
    c->scale = loss_scale; c->hyper = h; c->flags = flags;
    c->lay = make_layout(world, n_params);
    c->n_pad = c->lay.shard * world;
    if (const char* t = std::getenv("LMSGD_TIMEOUT_MS")) c->timeout_ns = std::atoll(t) * 1000000LL;
    DeviceGuard g(device);
    auto bail = [&](lmsgd_status s) { c->connected = false; lmsgd_finalize(c); return s; };
    if ((e = cudaMalloc(&c->buf, c->lay.bytes)) != cudaSuccess) { g_err = "cudaMalloc exchange buffer"; return bail(LMSGD_ERR_CUDA); }
    if ((e = cudaMemset(c->buf, 0, c->lay.bytes)) != cudaSuccess) { g_err = "cudaMemset"; return bail(LMSGD_ERR_CUDA); }
    int64_t init_status[2 * lmsgd::ST_WORDS] = {};
    for (int p = 0; p < 2; ++p) {
        init_status[p * lmsgd::ST_WORDS + lmsgd::ST_FIRST] = lmsgd::kNone;
        init_status[p * lmsgd::ST_WORDS + lmsgd::ST_G_FIRST] = lmsgd::kNone;
    }
    if ((e = cudaMemcpy(c->buf + c->lay.off_status, init_status, sizeof init_status, cudaMemcpyHostToDevice)) != cudaSuccess) {
        g_err = "cudaMemcpy status"; return bail(LMSGD_ERR_CUDA);
    }
    if ((e = cudaMalloc(&c->tickets, 4 * sizeof(unsigned int))) != cudaSuccess ||
        (e = cudaMemset(c->tickets, 0, 4 * sizeof(unsigned int))) != cudaSuccess ||
        (e = cudaMalloc(&c->dstate, sizeof(lmsgd_ctx::DevState))) != cudaSuccess ||
        (e = cudaMemset(c->dstate, 0, sizeof(lmsgd_ctx::DevState))) != cudaSuccess ||
        (e = cudaMalloc(&c->xctr, (4 + c->lay.nchunks) * sizeof(unsigned int))) != cudaSuccess ||
        (e = cudaMemset(c->xctr, 0, (4 + c->lay.nchunks) * sizeof(unsigned int))) != cudaSuccess ||
        (e = cudaMalloc(&c->last, sizeof(lmsgd_step_status))) != cudaSuccess ||
        (e = cudaMemset(c->last, 0, sizeof(lmsgd_step_status))) != cudaSuccess) {
        g_err = std::string("context allocations: ") + cudaGetErrorString(e);
        return bail(LMSGD_ERR_CUDA);
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) { g_err = cudaGetErrorString(e); return bail(LMSGD_ERR_CUDA); }
    c->L = launch_for_current_device();
    for (int p = 0; p < LMSGD_MAX_WORLD; ++p) c->peers.base[p] = nullptr;
    c->peers.base[rank] = c->buf;
    c->connected = (world == 1);
    *out = c;
    return LMSGD_OK;
}

lmsgd_status lmsgd_ipc_handle(lmsgd_ctx* c, uint8_t* out) {
    if (!c || !out) return fail(c, LMSGD_ERR_INVALID_ARG, "NULL argument");
    if (c->world == 1) return fail(c, LMSGD_ERR_STATE, "world == 1 has no peers");
    DeviceGuard g(c->device);
    cudaIpcMemHandle_t h;
    CK(c, cudaIpcGetMemHandle(&h, c->buf));
    static_assert(sizeof(h) == LMSGD_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(out, &h, sizeof h);
    return LMSGD_OK;
}

lmsgd_status lmsgd_connect(lmsgd_ctx* c, const uint8_t* handles) {
    if (!c || !handles) return fail(c, LMSGD_ERR_INVALID_ARG, "NULL argument");
    if (c->world == 1) return LMSGD_OK;
    if (c->connected) return fail(c, LMSGD_ERR_STATE, "already connected");
    DeviceGuard g(c->device);
    for (int p = 0; p < c->world; ++p) {
        if (p == c->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + p * LMSGD_IPC_HANDLE_BYTES, sizeof h);
        void* ptr = nullptr;
        CK(c, cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        c->peers.base[p] = static_cast<char*>(ptr);
    }
    c->connected = true;
    return LMSGD_OK;
}

lmsgd_status lmsgd_nvls_supported(int device, int* supported) {
    if (!supported) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "supported is NULL");
    *supported = 0;
    if (!drv().ok) return LMSGD_OK;
    CUdevice dev = 0;
    int v = 0;
    CKD(nullptr, drv().devGet(&dev, device));
    CKD(nullptr, drv().devAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    *supported = v;
    return LMSGD_OK;
}

lmsgd_status lmsgd_nvls_create(lmsgd_ctx* c, uint8_t* handle_out) {
    lmsgd_status st = nvls_pre(c);
    if (st != LMSGD_OK) return st;
    if (!handle_out) return fail(c, LMSGD_ERR_INVALID_ARG, "handle_out is NULL");
    if (c->rank != 0) return fail(c, LMSGD_ERR_STATE, "lmsgd_nvls_create is rank 0's call");
    if (c->nv.stage != 0) return fail(c, LMSGD_ERR_STATE, "NVLS already set up");
    DeviceGuard g(c->device);
    CK(c, cudaFree(nullptr));   // the device's primary context is current
    const Drv& d = drv();
    CUdevice dev = 0;
    CKD(c, d.devGet(&dev, c->device));
    int sup = 0;
    CKD(c, d.devAttr(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    if (!sup) return fail(c, LMSGD_ERR_UNSUPPORTED, "device does not support multicast objects");
    // size: the fp16 wire [n_pad], rounded up to the multicast and allocation granularities
    CUmulticastObjectProp mp = mc_prop(c->world, 2 * static_cast<size_t>(c->n_pad));
    size_t gm = 0, ga = 0;
    CKD(c, d.mcGran(&gm, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    CKD(c, d.memGran(&ga, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    const size_t gran = gm > ga ? gm : ga;
    mp.size = (mp.size + gran - 1) / gran * gran;
    CKD(c, d.mcCreate(&c->nv.mc, &mp));
    c->nv.size = mp.size;
    c->nv.stage = 1;
    int fd = -1;
    CKD(c, d.exportH(&fd, c->nv.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    c->nv.fd = fd;
    NvHandle h{};
    h.magic = kNvMagic;
    h.world = static_cast<uint32_t>(c->world);
    h.size = mp.size;
    timespec ts{};
    clock_gettime(CLOCK_MONOTONIC, &ts);
    std::snprintf(h.name, sizeof h.name, "lmsgd-nvls-%d-%llx", static_cast<int>(getpid()),
                  static_cast<unsigned long long>(ts.tv_sec * 1000000000LL + ts.tv_nsec));
    const int lfd = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    sockaddr_un a;
    const socklen_t al = abstract_addr(h.name, &a);
    if (lfd < 0 || bind(lfd, reinterpret_cast<sockaddr*>(&a), al) != 0 || listen(lfd, c->world) != 0) {
        if (lfd >= 0) close(lfd);
        return fail(c, LMSGD_ERR_CUDA, "NVLS: cannot listen on the fd-passing socket");
    }
    c->nv.server = std::thread(fd_server, lfd, fd, c->world - 1);
    std::memcpy(handle_out, &h, sizeof h);
    // rank 0 joins its own multicast object
    CKD(c, d.mcAdd(c->nv.mc, dev));
    return LMSGD_OK;
}

lmsgd_status lmsgd_nvls_connect(lmsgd_ctx* c, const uint8_t* handle) {
    lmsgd_status st = nvls_pre(c);
    if (st != LMSGD_OK) return st;
    if (!handle) return fail(c, LMSGD_ERR_INVALID_ARG, "handle is NULL");
    NvHandle h{};
    std::memcpy(&h, handle, sizeof h);
    if (h.magic != kNvMagic || h.world != static_cast<uint32_t>(c->world) || h.size < 2 * static_cast<uint64_t>(c->n_pad))
        return fail(c, LMSGD_ERR_INVALID_ARG, "NVLS handle does not match this context");
    if (c->rank == 0) return c->nv.stage == 1 ? LMSGD_OK : fail(c, LMSGD_ERR_STATE, "rank 0: call lmsgd_nvls_create first");
    if (c->nv.stage != 0) return fail(c, LMSGD_ERR_STATE, "NVLS already set up");
    DeviceGuard g(c->device);
    CK(c, cudaFree(nullptr));
    const Drv& d = drv();
    h.name[sizeof h.name - 1] = 0;
    const int fd = fd_fetch(h.name);
    if (fd < 0) return fail(c, LMSGD_ERR_CUDA, "NVLS: could not fetch the multicast fd from rank 0");
    c->nv.fd = fd;
    CKD(c, d.importH(&c->nv.mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                     CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    c->nv.size = h.size;
    c->nv.stage = 1;
    CUdevice dev = 0;
    CKD(c, d.devGet(&dev, c->device));
    CKD(c, d.mcAdd(c->nv.mc, dev));
    return LMSGD_OK;
}

lmsgd_status lmsgd_nvls_bind(lmsgd_ctx* c, int mode) {
    lmsgd_status st = nvls_pre(c);
    if (st != LMSGD_OK) return st;
    if (mode < LMSGD_NVLS_OFF || mode > LMSGD_NVLS_ALLREDUCE) return fail(c, LMSGD_ERR_INVALID_ARG, "bad NVLS mode");
    if (c->nv.stage != 1) return fail(c, LMSGD_ERR_STATE, "NVLS: lmsgd_nvls_connect first (and bind once)");
    DeviceGuard g(c->device);
    const Drv& d = drv();
    if (c->nv.server.joinable()) c->nv.server.join();   // every peer connected before the barrier
    CUdevice dev = 0;
    CKD(c, d.devGet(&dev, c->device));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    // "externally shareable as well as imported multicast objects can be bound only to
    // externally shareable memory" (cuda.h, cuMulticastBindMem)
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    const size_t size = c->nv.size;
    CKD(c, d.memCreate(&c->nv.phys, size, &ap, 0));
    CKD(c, d.mcBind(c->nv.mc, 0, c->nv.phys, 0, size, 0));
    c->nv.bound = true;
    // VA alignment: the larger of the allocation and multicast granularities (the size
    // is a multiple of both, lmsgd_nvls_create)
    size_t gran = 0, gm = 0;
    CKD(c, d.memGran(&gran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    const CUmulticastObjectProp mp = mc_prop(c->world, size);
    CKD(c, d.mcGran(&gm, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    gran = gm > gran ? gm : gran;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CKD(c, d.addrReserve(&c->nv.uc_va, size, gran, 0, 0));
    CKD(c, d.memMap(c->nv.uc_va, size, 0, c->nv.phys, 0));
    c->nv.uc_mapped = true;
    CKD(c, d.setAccess(c->nv.uc_va, size, &acc, 1));
    CKD(c, d.addrReserve(&c->nv.mc_va, size, gran, 0, 0));
    CKD(c, d.memMap(c->nv.mc_va, size, 0, c->nv.mc, 0));
    c->nv.mc_mapped = true;
    CKD(c, d.setAccess(c->nv.mc_va, size, &acc, 1));
    CK(c, cudaMemset(reinterpret_cast<void*>(c->nv.uc_va), 0, size));
    CK(c, cudaDeviceSynchronize());
    c->nv.stage = 2;
    c->nv.mode = mode;
    return LMSGD_OK;
}

lmsgd_status lmsgd_nvls_mode(lmsgd_ctx* c, int mode) {
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (mode < LMSGD_NVLS_OFF || mode > LMSGD_NVLS_ALLREDUCE) return fail(c, LMSGD_ERR_INVALID_ARG, "bad NVLS mode");
    if (mode != LMSGD_NVLS_OFF && c->nv.stage != 2) return fail(c, LMSGD_ERR_STATE, "NVLS is not bound");
    c->nv.mode = mode;
    return LMSGD_OK;
}

lmsgd_status lmsgd_finalize(lmsgd_ctx* c) {
    if (!c) return LMSGD_OK;
    {
        DeviceGuard g(c->device);
        cudaDeviceSynchronize();
        for (int p = 0; p < LMSGD_MAX_WORLD; ++p)
            if (!c->group && p != c->rank && c->peers.base[p]) cudaIpcCloseMemHandle(c->peers.base[p]);
        if (c->d_group) cudaFree(c->d_group);
        if (c->d_group_graph) cudaFree(c->d_group_graph);
        if (c->d_group_bn) cudaFree(c->d_group_bn);
        if (c->buf) cudaFree(c->buf);
        if (c->tickets) cudaFree(c->tickets);
        if (c->xctr) cudaFree(c->xctr);
        if (c->dstate) cudaFree(c->dstate);
        if (c->d_ctab) cudaFree(c->d_ctab);
        if (c->last) cudaFree(c->last);
        for (int b = 0; b < 2; ++b) {
            if (c->d_grads[b]) cudaFree(c->d_grads[b]);
            if (c->ev_copied[b]) cudaEventDestroy(c->ev_copied[b]);
            if (c->ev_consumed[b]) cudaEventDestroy(c->ev_consumed[b]);
        }
        if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
        if (c->d_trace) cudaFree(c->d_trace);
        nvls_release(c);
        for (auto& r : c->recs) { c->pool.push_back(r.a); c->pool.push_back(r.b); }
        for (auto e : c->pool) cudaEventDestroy(e);
    }
    delete c;
    return LMSGD_OK;
}

lmsgd_status lmsgd_step(lmsgd_ctx* c, void* stream, float* params, const float* grads, float* delta,
                        float* m, const lmsgd_coeffs* coeffs) {
    NvtxRange nvtx_("lmsgd_step");
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (!aligned16(params) || !aligned16(grads) || !aligned16(delta) || !aligned16(m))
        return fail(c, LMSGD_ERR_INVALID_ARG, "params/grads/delta/m must be non-NULL and 16-byte aligned");
    if (!coeffs_ok(coeffs))
        return fail(c, LMSGD_ERR_INVALID_ARG, "coeffs: need eta > 0, 0 <= alpha_sgd <= 1, alpha_rmsprop >= 0");
    if (!c->connected) return fail(c, LMSGD_ERR_STATE, "lmsgd_connect has not been called");
    if (c->group) return fail(c, LMSGD_ERR_STATE, "group-connected context: use the lmsgd_*_group calls");
    if (c->mode == 2) return fail(c, LMSGD_ERR_STATE, "this context already runs lmsgd_step_graph");
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    UpdConst u = make_const(c->hyper, *coeffs, c->world, c->scale, c->wd, c->n_wd);
    u.freeze_m = (c->flags & LMSGD_FLAG_FREEZE_M) && u.a_rms == 0.0f;
    const uint32_t epoch = ++c->step;
    const int parity = static_cast<int>(epoch & 1u);
    c->last_stream = s;
    c->mode = 1;
    if (c->world == 1) {
        uint16_t* h = reinterpret_cast<uint16_t*>(c->buf + c->lay.off_recv);
        if (c->flags & LMSGD_FLAG_NO_SKIP) {
            CK(c, timed(c, s, 0, [&] {
                   return lmsgd::launch_fused1(s, c->L, grads, c->n, c->scale, u, params, delta, m,
                                               status_slot(c, parity), status_slot(c, parity ^ 1), nullptr);
               }));
            CK(c, lmsgd::launch_finalize_fused(s, status_slot(c, parity), c->last));
        } else {
            CK(c, timed(c, s, 0, [&] {
                   return lmsgd::launch_pack(s, c->L, grads, c->n, c->n_pad, c->scale, h, status_slot(c, parity));
               }));
            CK(c, timed(c, s, 2, [&] {
                   return lmsgd::launch_update(s, c->L, h, c->n, u, params, delta, m, status_slot(c, parity),
                                               status_slot(c, parity ^ 1), c->last);
               }));
        }
        return LMSGD_OK;
    }
    const lmsgd::XArgs x = xargs(c, epoch, &c->dstate->xepoch);
    lmsgd::XStep a{x, grads, c->scale, u, params, delta, m, c->last, c->xctr, nullptr, 0, nullptr};
    a.v8 = 1;   // 256-bit accesses if params / delta / m are 32-byte aligned (launch_xstep checks)
    a.riu = 1;  // own-shard reduce inside the update (kernels.cu riu_active)
    CK(c, timed(c, s, 2, [&] { return lmsgd::launch_xstep(s, xlaunch(c), a); }));
    return LMSGD_OK;
}

lmsgd_status lmsgd_step_out_of_place(lmsgd_ctx* c, void* stream, const float* params_in, float* params_out,
                                      const float* grads, const float* delta_in, float* delta_out,
                                      const float* m_in, float* m_out, const lmsgd_coeffs* coeffs) {
    NvtxRange nvtx_("lmsgd_step_out_of_place");
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (!aligned16(params_in) || !aligned16(params_out) || !aligned16(grads) || !aligned16(delta_in) ||
        !aligned16(delta_out) || !aligned16(m_in) || !aligned16(m_out))
        return fail(c, LMSGD_ERR_INVALID_ARG, "all pointers must be non-NULL and 16-byte aligned");
    const int64_t bytes = c->n * 4;
    auto overlap = [&](const void* a, const void* b) {
        const char* x = static_cast<const char*>(a);
        const char* y = static_cast<const char*>(b);
        return x < y + bytes && y < x + bytes;
    };
    const void* ins[] = {params_in, delta_in, m_in, grads};
    const void* outs[] = {params_out, delta_out, m_out};
    for (const void* o : outs)
        for (const void* i : ins)
            if (overlap(o, i)) return fail(c, LMSGD_ERR_INVALID_ARG, "output buffers must not overlap the inputs");
    if (!coeffs_ok(coeffs))
        return fail(c, LMSGD_ERR_INVALID_ARG, "coeffs: need eta > 0, 0 <= alpha_sgd <= 1, alpha_rmsprop >= 0");
    if (c->world != 1) return fail(c, LMSGD_ERR_UNSUPPORTED, "out-of-place step is world == 1 only (use lmsgd_step)");
    if (c->wd != 0.0) return fail(c, LMSGD_ERR_UNSUPPORTED, "out-of-place step has no weight decay");
    if (c->flags != 0)
        return fail(c, LMSGD_ERR_UNSUPPORTED, "out-of-place step: a context created with flags (NO_SKIP / FREEZE_M)");
    if (c->mode == 2) return fail(c, LMSGD_ERR_STATE, "this context runs lmsgd_step_graph");
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const UpdConst u = make_const(c->hyper, *coeffs, 1, c->scale, 0.0, 0);
    const uint32_t epoch = ++c->step;
    const int parity = static_cast<int>(epoch & 1u);
    c->last_stream = s;
    c->mode = 1;
    int64_t* trace = nullptr;   // lmsgd_trace_enable: the kernel's start and end stamps
    if (c->d_trace) {
        trace = c->d_trace + (c->trace_steps % c->trace_cap) * lmsgd::TR_WORDS;
        ++c->trace_steps;
    }
    CK(c, timed(c, s, 0, [&] {
           return lmsgd::launch_step_oop1(s, c->L, grads, c->n, c->scale, u, params_in, delta_in, m_in, params_out,
                                          delta_out, m_out, status_slot(c, parity), status_slot(c, parity ^ 1),
                                          c->last, trace);
       }));
    return LMSGD_OK;
}

lmsgd_status lmsgd_exchange(lmsgd_ctx* c, void* stream, const float* grads, uint16_t* R_out) {
    NvtxRange nvtx_("lmsgd_exchange");
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (!aligned16(grads) || !aligned16(R_out))
        return fail(c, LMSGD_ERR_INVALID_ARG, "grads/R_out must be non-NULL and 16-byte aligned");
    if (!c->connected) return fail(c, LMSGD_ERR_STATE, "lmsgd_connect has not been called");
    if (c->group) return fail(c, LMSGD_ERR_STATE, "group-connected context: use the lmsgd_*_group calls");
    if (c->mode == 2) return fail(c, LMSGD_ERR_STATE, "this context runs lmsgd_step_graph");
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t epoch = ++c->step;   // one collective epoch, shared with lmsgd_step
    const int parity = static_cast<int>(epoch & 1u);
    c->last_stream = s;
    c->mode = 1;   // host-mode epochs and status slots, like lmsgd_step (not mixed with graph mode)
    if (c->world == 1) {
        CK(c, timed(c, s, 0, [&] {
               return lmsgd::launch_pack(s, c->L, grads, c->n, c->n_pad, c->scale, R_out, status_slot(c, parity));
           }));
        CK(c, lmsgd::launch_xfinal1(s, status_slot(c, parity), status_slot(c, parity ^ 1), c->last));
        return LMSGD_OK;
    }
    const lmsgd::XArgs x = xargs(c, epoch, &c->dstate->xepoch);
    lmsgd::XStep a{x, grads, c->scale, lmsgd::UpdConst{}, nullptr, nullptr, nullptr, c->last, c->xctr,
                   nullptr, 0, nullptr, R_out};
    CK(c, timed(c, s, 2, [&] { return lmsgd::launch_xstep(s, xlaunch(c), a); }));
    return LMSGD_OK;
}

lmsgd_status lmsgd_status_accumulate(lmsgd_ctx* c, void* stream, int64_t offset, int64_t* dstatus) {
    if (!c || !dstatus || offset < 0) return fail(c, LMSGD_ERR_INVALID_ARG, "status_accumulate: bad argument");
    if (c->step == 0) return fail(c, LMSGD_ERR_STATE, "no exchange or step has run on this context");
    DeviceGuard g(c->device);
    CK(c, lmsgd::launch_status_accumulate(static_cast<cudaStream_t>(stream), c->last, offset, dstatus));
    return LMSGD_OK;
}

lmsgd_status lmsgd_set_exchange_blocks(lmsgd_ctx* c, int blocks) {
    if (!c || blocks < 0) return fail(c, LMSGD_ERR_INVALID_ARG, "set_exchange_blocks: bad argument");
    c->xblocks = blocks;
    return LMSGD_OK;
}

lmsgd_status lmsgd_set_weight_decay(lmsgd_ctx* c, double lambda, int64_t n_decay) {
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (!(lambda >= 0.0) || !std::isfinite(lambda) || n_decay < -1 || n_decay > c->n)
        return fail(c, LMSGD_ERR_INVALID_ARG, "weight decay: need lambda >= 0 and -1 <= n_decay <= n_params");
    c->wd = lambda;
    c->n_wd = n_decay < 0 ? c->n : n_decay;
    return LMSGD_OK;
}

lmsgd_status lmsgd_schedule_upload(lmsgd_ctx* c, const lmsgd_hyper* hyper, const lmsgd_cluster* cluster,
                                   int64_t t_first, int64_t count) {
    if (!c || !cluster || t_first < 1 || count < 1 || count > (int64_t(1) << 24))
        return fail(c, LMSGD_ERR_INVALID_ARG, "schedule_upload: bad argument");
    lmsgd_hyper h{};
    if (hyper) h = *hyper; else lmsgd_hyper_default(&h);
    std::vector<UpdConst> tab(static_cast<size_t>(count));
    for (int64_t i = 0; i < count; ++i) {
        lmsgd_coeffs co{};
        const lmsgd_status st = lmsgd_schedule_at(&h, cluster, t_first + i, &co);
        if (st != LMSGD_OK) return fail(c, st, "schedule_upload: step " + std::to_string(t_first + i) + " is out of range");
        tab[static_cast<size_t>(i)] = make_const(c->hyper, co, c->world, c->scale, c->wd, c->n_wd);
    }
    DeviceGuard g(c->device);
    CK(c, cudaDeviceSynchronize());
    if (count > c->ctab_cap) {
        if (c->d_ctab) cudaFree(c->d_ctab);
        c->d_ctab = nullptr;
        CK(c, cudaMalloc(&c->d_ctab, count * sizeof(UpdConst)));
        c->ctab_cap = count;
    }
    CK(c, cudaMemcpy(c->d_ctab, tab.data(), count * sizeof(UpdConst), cudaMemcpyHostToDevice));
    CK(c, cudaMemset(&c->dstate->cursor, 0, sizeof(int64_t)));
    c->ctab_count = count;
    c->ctab_n_wd = tab[0].n_wd;
    return LMSGD_OK;
}

lmsgd_status lmsgd_step_graph(lmsgd_ctx* c, void* stream, float* params, const float* grads, float* delta,
                              float* m) {
    NvtxRange nvtx_("lmsgd_step_graph");
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (!aligned16(params) || !aligned16(grads) || !aligned16(delta) || !aligned16(m))
        return fail(c, LMSGD_ERR_INVALID_ARG, "params/grads/delta/m must be non-NULL and 16-byte aligned");
    if (!c->connected) return fail(c, LMSGD_ERR_STATE, "lmsgd_connect has not been called");
    if (c->group) return fail(c, LMSGD_ERR_STATE, "group-connected context: use the lmsgd_*_group calls");
    if (c->ctab_count == 0) return fail(c, LMSGD_ERR_STATE, "lmsgd_schedule_upload has not been called");
    if (c->mode == 1) return fail(c, LMSGD_ERR_STATE, "this context already runs lmsgd_step / lmsgd_exchange");
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    UpdConst u{};         // every coefficient comes from the device table; n_wd selects the kernel variant
    u.n_wd = c->ctab_n_wd;
    c->last_stream = s;
    ++c->step;            // host-side count only (the kernels use the device counter)
    c->mode = 2;
    if (c->world == 1) {
        lmsgd::Dev1 dv{&c->dstate->k1epoch, status_slot(c, 0), c->d_ctab, c->ctab_count, &c->dstate->cursor};
        uint16_t* h = reinterpret_cast<uint16_t*>(c->buf + c->lay.off_recv);
        if (c->flags & LMSGD_FLAG_NO_SKIP) {
            CK(c, lmsgd::launch_fused1(s, c->L, grads, c->n, c->scale, u, params, delta, m, nullptr, nullptr,
                                       nullptr, dv));
            CK(c, lmsgd::launch_advance1(s, dv, c->last, true));
        } else {
            CK(c, lmsgd::launch_pack(s, c->L, grads, c->n, c->n_pad, c->scale, h, nullptr, dv));
            CK(c, lmsgd::launch_update(s, c->L, h, c->n, u, params, delta, m, nullptr, nullptr, c->last, dv));
            CK(c, lmsgd::launch_advance1(s, dv, c->last, false));
        }
        return LMSGD_OK;
    }
    lmsgd::XArgs x = xargs(c, 0, &c->dstate->xepoch);
    if (x.trace) { x.trace = nullptr; --c->trace_steps; }   // the trace ring slot would be frozen in a graph
    lmsgd::XStep a{x, grads, c->scale, u, params, delta, m, c->last, c->xctr, c->d_ctab, c->ctab_count,
                   &c->dstate->cursor};
    a.v8 = 1;
    a.riu = 1;
    CK(c, lmsgd::launch_xstep(s, xlaunch(c), a));
    return LMSGD_OK;
}

namespace {
// Host->device copy of this step's gradient into one of two device staging buffers on
// the library's copy stream; `stream` waits for it.  Returns the staging buffer.
lmsgd_status stage_grads(lmsgd_ctx* c, cudaStream_t s, const float* grads_host, int* b_out) {
    if (!c->copy_stream) {
        CK(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CK(c, cudaMalloc(&c->d_grads[b], c->n * sizeof(float)));
            CK(c, cudaEventCreateWithFlags(&c->ev_copied[b], cudaEventDisableTiming));
            CK(c, cudaEventCreateWithFlags(&c->ev_consumed[b], cudaEventDisableTiming));
            CK(c, cudaEventRecord(c->ev_consumed[b], c->copy_stream));
        }
    }
    const int b = c->host_buf;
    c->host_buf ^= 1;
    // buffer b is free once the step that last read it has passed on its stream
    CK(c, cudaStreamWaitEvent(c->copy_stream, c->ev_consumed[b], 0));
    CK(c, cudaMemcpyAsync(c->d_grads[b], grads_host, c->n * sizeof(float), cudaMemcpyHostToDevice, c->copy_stream));
    CK(c, cudaEventRecord(c->ev_copied[b], c->copy_stream));
    CK(c, cudaStreamWaitEvent(s, c->ev_copied[b], 0));
    *b_out = b;
    return LMSGD_OK;
}

// After the step on `s`: staging buffer b is free again; the step's parameters (if
// params_host) and status record go back to the host on `s`.
lmsgd_status finish_host_step(lmsgd_ctx* c, cudaStream_t s, int b, const float* params_dev, float* params_host,
                              lmsgd_step_status* status_host) {
    CK(c, cudaEventRecord(c->ev_consumed[b], s));
    if (params_host)
        CK(c, cudaMemcpyAsync(params_host, params_dev, c->n * sizeof(float), cudaMemcpyDeviceToHost, s));
    CK(c, cudaMemcpyAsync(status_host, c->last, sizeof(lmsgd_step_status), cudaMemcpyDeviceToHost, s));
    return LMSGD_OK;
}
}  // namespace

lmsgd_status lmsgd_step_host(lmsgd_ctx* c, void* stream, float* params, const float* grads_host,
                             float* delta, float* m, const lmsgd_coeffs* coeffs, float* params_host,
                             lmsgd_step_status* status_host) {
    NvtxRange nvtx_("lmsgd_step_host");
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (!grads_host || !status_host) return fail(c, LMSGD_ERR_INVALID_ARG, "NULL host pointer");
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int b = 0;
    lmsgd_status st = stage_grads(c, s, grads_host, &b);
    if (st != LMSGD_OK) return st;
    st = lmsgd_step(c, stream, params, c->d_grads[b], delta, m, coeffs);
    if (st != LMSGD_OK) return st;
    return finish_host_step(c, s, b, params, params_host, status_host);
}

lmsgd_status lmsgd_step_out_of_place_host(lmsgd_ctx* c, void* stream, const float* params_in, float* params_out,
                                          const float* grads_host, const float* delta_in, float* delta_out,
                                          const float* m_in, float* m_out, const lmsgd_coeffs* coeffs,
                                          float* params_host, lmsgd_step_status* status_host) {
    NvtxRange nvtx_("lmsgd_step_out_of_place_host");
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (!grads_host || !status_host) return fail(c, LMSGD_ERR_INVALID_ARG, "NULL host pointer");
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int b = 0;
    lmsgd_status st = stage_grads(c, s, grads_host, &b);
    if (st != LMSGD_OK) return st;
    st = lmsgd_step_out_of_place(c, stream, params_in, params_out, c->d_grads[b], delta_in, delta_out, m_in, m_out,
                                 coeffs);
    if (st != LMSGD_OK) return st;
    return finish_host_step(c, s, b, params_out, params_host, status_host);
}

lmsgd_status lmsgd_query_status(lmsgd_ctx* c, lmsgd_step_status* out) {
    if (!c || !out) return fail(c, LMSGD_ERR_INVALID_ARG, "NULL argument");
    if (c->step == 0) return fail(c, LMSGD_ERR_STATE, "no step has run");
    DeviceGuard g(c->device);
    CK(c, cudaStreamSynchronize(c->last_stream));
    CK(c, cudaMemcpy(out, c->last, sizeof *out, cudaMemcpyDeviceToHost));
    if (out->error != 0) return static_cast<lmsgd_status>(out->error);
    return LMSGD_OK;
}

lmsgd_status lmsgd_bn_stats_allreduce(lmsgd_ctx* c, void* stream, float* mean, float* var, int64_t C) {
    NvtxRange nvtx_("lmsgd_bn_stats_allreduce");
    if (!c) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "ctx is NULL");
    if (!mean || !var || C < 1 || C > LMSGD_MAX_BN_CHANNELS)
        return fail(c, LMSGD_ERR_INVALID_ARG, "mean/var must be non-NULL, 0 < C <= LMSGD_MAX_BN_CHANNELS");
    if (!c->connected) return fail(c, LMSGD_ERR_STATE, "lmsgd_connect has not been called");
    if (c->group) return fail(c, LMSGD_ERR_STATE, "group-connected context: use the lmsgd_*_group calls");
    if (c->world == 1) return LMSGD_OK;  // the average of one worker is itself
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ++c->bn_calls;
    lmsgd::XArgs x = xargs(c, 0, &c->dstate->bnepoch);   // epoch from the device call counter
    if (x.trace) { x.trace = nullptr; --c->trace_steps; }
    CK(c, lmsgd::launch_bn_allreduce(s, lmsgd::BnArgs{x, mean, var, C}));
    return LMSGD_OK;
}

lmsgd_status lmsgd_profile_enable(lmsgd_ctx* c, int64_t max_launches) {
    if (!c || max_launches < 0 || max_launches > (int64_t(1) << 22))
        return fail(c, LMSGD_ERR_INVALID_ARG, "profile_enable: bad argument");
    DeviceGuard g(c->device);
    CK(c, cudaDeviceSynchronize());
    for (auto& r : c->recs) { c->pool.push_back(r.a); c->pool.push_back(r.b); }
    c->recs.clear();
    c->prof_cap = static_cast<size_t>(max_launches);
    while (c->pool.size() < 2 * c->prof_cap) {
        cudaEvent_t e;
        CK(c, cudaEventCreate(&e));
        c->pool.push_back(e);
    }
    return LMSGD_OK;
}

lmsgd_status lmsgd_profile_read(lmsgd_ctx* c, double* ms, int64_t* launches) {
    if (!c || !ms || !launches) return fail(c, LMSGD_ERR_INVALID_ARG, "profile_read: NULL argument");
    DeviceGuard g(c->device);
    for (int p = 0; p < 3; ++p) { ms[p] = 0.0; launches[p] = 0; }
    for (auto& r : c->recs) {
        CK(c, cudaEventSynchronize(r.b));
        float t = 0.0f;
        CK(c, cudaEventElapsedTime(&t, r.a, r.b));
        ms[r.phase] += t;
        launches[r.phase] += 1;
        c->pool.push_back(r.a);
        c->pool.push_back(r.b);
    }
    c->recs.clear();
    return LMSGD_OK;
}

lmsgd_status lmsgd_trace_enable(lmsgd_ctx* c, int64_t max_steps) {
    if (!c || max_steps < 0 || max_steps > (int64_t(1) << 20))
        return fail(c, LMSGD_ERR_INVALID_ARG, "trace_enable: bad argument");
    DeviceGuard g(c->device);
    CK(c, cudaDeviceSynchronize());
    if (c->d_trace) { cudaFree(c->d_trace); c->d_trace = nullptr; }
    c->trace_cap = max_steps;
    c->trace_steps = 0;
    if (max_steps > 0) {
        CK(c, cudaMalloc(&c->d_trace, max_steps * lmsgd::TR_WORDS * sizeof(int64_t)));
        CK(c, cudaMemset(c->d_trace, 0, max_steps * lmsgd::TR_WORDS * sizeof(int64_t)));
    }
    return LMSGD_OK;
}

lmsgd_status lmsgd_trace_read(lmsgd_ctx* c, int64_t* out, int64_t max_steps, int64_t* steps) {
    if (!c || !out || !steps || max_steps < 0) return fail(c, LMSGD_ERR_INVALID_ARG, "trace_read: bad argument");
    DeviceGuard g(c->device);
    CK(c, cudaDeviceSynchronize());
    const int64_t have = c->trace_steps < c->trace_cap ? c->trace_steps : c->trace_cap;
    *steps = have < max_steps ? have : max_steps;
    if (*steps > 0)
        CK(c, cudaMemcpy(out, c->d_trace, *steps * lmsgd::TR_WORDS * sizeof(int64_t), cudaMemcpyDeviceToHost));
    return LMSGD_OK;
}

// ---------------------------------------------------------------- emulated groups
// The ranks of a world as contexts of ONE process on ONE GPU, connected in-process and
// stepped together: each kernel of the world > 1 path is launched once for all of
// them (the SIM instantiations), so ranks that wait for one another are co-scheduled.


lmsgd_status lmsgd_connect_group(lmsgd_ctx* const* ctxs, int world) {
    lmsgd_status st = group_check(ctxs, world, false);
    if (st != LMSGD_OK) return st;
    if (world != ctxs[0]->world) return fail(ctxs[0], LMSGD_ERR_INVALID_ARG, "connect_group: need all world ranks");
    for (int i = 0; i < world; ++i)
        if (ctxs[i]->connected) return fail(ctxs[i], LMSGD_ERR_STATE, "connect_group: already connected");
    for (int i = 0; i < world; ++i) {
        lmsgd_ctx* c = ctxs[i];
        for (int j = 0; j < world; ++j) c->peers.base[ctxs[j]->rank] = ctxs[j]->buf;
        c->group = true;
        c->connected = true;
    }
    return LMSGD_OK;
}

lmsgd_status lmsgd_step_group(lmsgd_ctx* const* ctxs, int count, void* stream, float* const* params,
                              const float* const* grads, float* const* delta, float* const* m,
                              const lmsgd_coeffs* coeffs) {
    NvtxRange nvtx_("lmsgd_step_group");
    lmsgd_status st = group_check(ctxs, count, true);
    if (st != LMSGD_OK) return st;
    if (!params || !grads || !delta || !m) return fail(ctxs[0], LMSGD_ERR_INVALID_ARG, "group step: NULL array");
    if (!coeffs_ok(coeffs))
        return fail(ctxs[0], LMSGD_ERR_INVALID_ARG, "coeffs: need eta > 0, 0 <= alpha_sgd <= 1, alpha_rmsprop >= 0");
    for (int i = 0; i < count; ++i) {
        if (!aligned16(params[i]) || !aligned16(grads[i]) || !aligned16(delta[i]) || !aligned16(m[i]))
            return fail(ctxs[i], LMSGD_ERR_INVALID_ARG, "params/grads/delta/m must be non-NULL and 16-byte aligned");
        if (ctxs[i]->mode == 2) return fail(ctxs[i], LMSGD_ERR_STATE, "this context runs lmsgd_step_graph_group");
    }
    lmsgd_ctx* lead = ctxs[0];
    DeviceGuard g(lead->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<lmsgd::XStep> v(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) {
        lmsgd_ctx* c = ctxs[i];
        UpdConst u = make_const(c->hyper, *coeffs, c->world, c->scale, c->wd, c->n_wd);
        u.freeze_m = (c->flags & LMSGD_FLAG_FREEZE_M) && u.a_rms == 0.0f;
        const uint32_t epoch = ++c->step;
        c->last_stream = s;
        c->mode = 1;
        v[i] = lmsgd::XStep{xargs(c, epoch, &c->dstate->xepoch), grads[i], c->scale, u, params[i], delta[i], m[i],
                            c->last, c->xctr, nullptr, 0, nullptr, nullptr};
        v[i].riu = 1;
    }
    set_group_v8(v);
    if ((st = group_upload(lead, s, &lead->d_group, v)) != LMSGD_OK) return st;
    CK(lead, lmsgd::launch_xstep(s, lead->L, v[0], lead->d_group, count));
    return LMSGD_OK;
}

lmsgd_status lmsgd_exchange_group(lmsgd_ctx* const* ctxs, int count, void* stream, const float* const* grads,
                                  uint16_t* const* R_out) {
    NvtxRange nvtx_("lmsgd_exchange_group");
    lmsgd_status st = group_check(ctxs, count, true);
    if (st != LMSGD_OK) return st;
    if (!grads || !R_out) return fail(ctxs[0], LMSGD_ERR_INVALID_ARG, "group exchange: NULL array");
    for (int i = 0; i < count; ++i) {
        if (!aligned16(grads[i]) || !aligned16(R_out[i]))
            return fail(ctxs[i], LMSGD_ERR_INVALID_ARG, "grads/R_out must be non-NULL and 16-byte aligned");
        if (ctxs[i]->mode == 2) return fail(ctxs[i], LMSGD_ERR_STATE, "this context runs lmsgd_step_graph_group");
    }
    lmsgd_ctx* lead = ctxs[0];
    DeviceGuard g(lead->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<lmsgd::XStep> v(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) {
        lmsgd_ctx* c = ctxs[i];
        const uint32_t epoch = ++c->step;
        c->last_stream = s;
        c->mode = 1;
        v[i] = lmsgd::XStep{xargs(c, epoch, &c->dstate->xepoch), grads[i], c->scale, lmsgd::UpdConst{}, nullptr,
                            nullptr, nullptr, c->last, c->xctr, nullptr, 0, nullptr, R_out[i]};
    }
    if ((st = group_upload(lead, s, &lead->d_group, v)) != LMSGD_OK) return st;
    CK(lead, lmsgd::launch_xstep(s, lead->L, v[0], lead->d_group, count));
    return LMSGD_OK;
}

lmsgd_status lmsgd_step_graph_group(lmsgd_ctx* const* ctxs, int count, void* stream, float* const* params,
                                    const float* const* grads, float* const* delta, float* const* m) {
    NvtxRange nvtx_("lmsgd_step_graph_group");
    lmsgd_status st = group_check(ctxs, count, true);
    if (st != LMSGD_OK) return st;
    if (!params || !grads || !delta || !m) return fail(ctxs[0], LMSGD_ERR_INVALID_ARG, "group step: NULL array");
    for (int i = 0; i < count; ++i) {
        lmsgd_ctx* c = ctxs[i];
        if (!aligned16(params[i]) || !aligned16(grads[i]) || !aligned16(delta[i]) || !aligned16(m[i]))
            return fail(c, LMSGD_ERR_INVALID_ARG, "params/grads/delta/m must be non-NULL and 16-byte aligned");
        if (c->ctab_count == 0) return fail(c, LMSGD_ERR_STATE, "lmsgd_schedule_upload has not been called");
        if (c->mode == 1) return fail(c, LMSGD_ERR_STATE, "this context already runs host-mode group calls");
    }
    lmsgd_ctx* lead = ctxs[0];
    DeviceGuard g(lead->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<lmsgd::XStep> v(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) {
        lmsgd_ctx* c = ctxs[i];
        UpdConst u{};
        u.n_wd = c->ctab_n_wd;
        c->last_stream = s;
        ++c->step;
        c->mode = 2;
        lmsgd::XArgs x = xargs(c, 0, &c->dstate->xepoch);
        if (x.trace) { x.trace = nullptr; --c->trace_steps; }
        v[i] = lmsgd::XStep{x, grads[i], c->scale, u, params[i], delta[i], m[i], c->last, c->xctr, c->d_ctab,
                            c->ctab_count, &c->dstate->cursor, nullptr};
        v[i].riu = 1;
    }
    set_group_v8(v);
    // the arguments do not change between graph-mode calls (everything per-step is read
    // from the device): upload once, outside any capture; a capture then records launches only
    const bool same = lead->group_graph_cache.size() == v.size() &&
                      std::memcmp(lead->group_graph_cache.data(), v.data(), v.size() * sizeof(lmsgd::XStep)) == 0;
    if (!same) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CK(lead, cudaStreamIsCapturing(s, &cs));
        if (cs != cudaStreamCaptureStatusNone)
            return fail(lead, LMSGD_ERR_STATE, "graph group: call once outside capture with these buffers first");
        if (!lead->d_group_graph) CK(lead, cudaMalloc(&lead->d_group_graph, LMSGD_MAX_WORLD * sizeof(lmsgd::XStep)));
        CK(lead, cudaStreamSynchronize(s));
        CK(lead, cudaMemcpy(lead->d_group_graph, v.data(), v.size() * sizeof(lmsgd::XStep), cudaMemcpyHostToDevice));
        lead->group_graph_cache = v;
    }
    CK(lead, lmsgd::launch_xstep(s, lead->L, v[0], lead->d_group_graph, count));
    return LMSGD_OK;
}

lmsgd_status lmsgd_bn_stats_allreduce_group(lmsgd_ctx* const* ctxs, int count, void* stream, float* const* mean,
                                            float* const* var, int64_t C) {
    NvtxRange nvtx_("lmsgd_bn_stats_allreduce_group");
    lmsgd_status st = group_check(ctxs, count, true);
    if (st != LMSGD_OK) return st;
    if (!mean || !var || C < 1 || C > LMSGD_MAX_BN_CHANNELS)
        return fail(ctxs[0], LMSGD_ERR_INVALID_ARG, "mean/var must be non-NULL, 0 < C <= LMSGD_MAX_BN_CHANNELS");
    lmsgd_ctx* lead = ctxs[0];
    DeviceGuard g(lead->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<lmsgd::BnArgs> v(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) {
        lmsgd_ctx* c = ctxs[i];
        if (!mean[i] || !var[i]) return fail(c, LMSGD_ERR_INVALID_ARG, "mean/var must be non-NULL");
        ++c->bn_calls;
        lmsgd::XArgs x = xargs(c, 0, &c->dstate->bnepoch);
        if (x.trace) { x.trace = nullptr; --c->trace_steps; }
        v[i] = lmsgd::BnArgs{x, mean[i], var[i], C};
    }
    if ((st = group_upload(lead, s, &lead->d_group_bn, v)) != LMSGD_OK) return st;
    CK(lead, lmsgd::launch_bn_allreduce(s, v[0], lead->d_group_bn, count));
    return LMSGD_OK;
}

// ---------------------------------------------------------------- sub-steps

lmsgd_status lmsgd_status_reset(void* stream, int64_t* dstatus) {
    if (!dstatus) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "dstatus is NULL");
    cudaError_t e = lmsgd::launch_status_reset(static_cast<cudaStream_t>(stream), dstatus);
    return e == cudaSuccess ? LMSGD_OK : cuda_fail(nullptr, e, "status_reset");
}

lmsgd_status lmsgd_pack(void* stream, const float* g, int64_t n, int64_t n_pad, float loss_scale,
                        uint16_t* h, int64_t* dstatus) {
    if (!aligned16(g) || !aligned16(h) || !dstatus || n < 0 || n_pad < n || n_pad % 8 != 0 || n_pad < 8)
        return fail(nullptr, LMSGD_ERR_INVALID_ARG, "pack: bad pointer or size (n_pad >= n, n_pad % 8 == 0)");
    if (!pow2_scale(loss_scale)) return fail(nullptr, LMSGD_ERR_INVALID_ARG, "loss_scale must be a power of two");
    cudaError_t e = lmsgd::launch_pack(static_cast<cudaStream_t>(stream), launch_for_current_device(), g, n,
                                       n_pad, loss_scale, h, dstatus);
    return e == cudaSuccess ? LMSGD_OK : cuda_fail(nullptr, e, "pack");
}

lmsgd_status lmsgd_reduce_local(void* stream, const uint16_t* h, int k, int64_t n_pad, uint16_t* R,
                                int64_t* dstatus) {
    if (!aligned16(h) || !aligned16(R) || k < 1 || k > 8192 || n_pad < 8 || n_pad % 8 != 0)
        return fail(nullptr, LMSGD_ERR_INVALID_ARG, "reduce_local: bad pointer, k or n_pad");
    cudaError_t e = lmsgd::launch_reduce_local(static_cast<cudaStream_t>(stream), launch_for_current_device(),
                                               h, k, n_pad, R, dstatus);
    return e == cudaSuccess ? LMSGD_OK : cuda_fail(nullptr, e, "reduce_local");
}

lmsgd_status lmsgd_update(void* stream, const uint16_t* R, int64_t n, int k, float loss_scale,
                          const lmsgd_hyper* hyper, const lmsgd_coeffs* coeffs, float* params, float* delta,
                          float* m, const int64_t* dstatus) {
    lmsgd_hyper h{};
    if (hyper) h = *hyper; else lmsgd_hyper_default(&h);
    if (!aligned16(R) || !aligned16(params) || !aligned16(delta) || !aligned16(m) || n < 1 || k < 1 ||
        !pow2_scale(loss_scale) || !hyper_ok(&h) || !coeffs_ok(coeffs))
        return fail(nullptr, LMSGD_ERR_INVALID_ARG, "update: bad pointer, size, scale, hyper or coeffs");
    const UpdConst u = make_const(h, *coeffs, k, loss_scale);
    cudaError_t e = lmsgd::launch_update(static_cast<cudaStream_t>(stream), launch_for_current_device(), R, n, u,
                                         params, delta, m, dstatus, nullptr, nullptr);
    return e == cudaSuccess ? LMSGD_OK : cuda_fail(nullptr, e, "update");
}

lmsgd_status lmsgd_fused_step1(void* stream, const float* g, int64_t n, float loss_scale,
                               const lmsgd_hyper* hyper, const lmsgd_coeffs* coeffs, float* params,
                               float* delta, float* m, int64_t* dstatus) {
    lmsgd_hyper h{};
    if (hyper) h = *hyper; else lmsgd_hyper_default(&h);
    if (!aligned16(g) || !aligned16(params) || !aligned16(delta) || !aligned16(m) || !dstatus || n < 1 ||
        !pow2_scale(loss_scale) || !hyper_ok(&h) || !coeffs_ok(coeffs))
        return fail(nullptr, LMSGD_ERR_INVALID_ARG, "fused_step1: bad pointer, size, scale, hyper or coeffs");
    const UpdConst u = make_const(h, *coeffs, 1, loss_scale);
    cudaError_t e = lmsgd::launch_fused1(static_cast<cudaStream_t>(stream), launch_for_current_device(), g, n,
                                         loss_scale, u, params, delta, m, dstatus, nullptr, nullptr);
    return e == cudaSuccess ? LMSGD_OK : cuda_fail(nullptr, e, "fused_step1");
}

}  // extern "C"
