// capi.cu - the extern "C" boundary (include/dotg.h): argument validation with the
// reference's error cases, device checks, dispatch to the kernels, and the host-buffer
// pipelines (copy / compute overlap on two streams).
//
// Error mapping (reference throws std::invalid_argument):
//   span length mismatch          addsub.cpp:139-140   -> not expressible (one m)
//   mul m == 0 / m > 2^24         mul.cpp:13-18        -> DOTG_EINVAL
//   unknown width                 addsub.cpp:125-134   -> dotg_validate_width
//   partial aliasing              undefined in ref     -> DOTG_EINVAL (stricter)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dotg.h"
#include "internal.h"

namespace dotg {
std::atomic<uint64_t> g_launches{0};
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(DOTG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// The device path is sm_100a-only; refuse anything else loudly (no CPU fallback).
int check_device() {
    // Start every call with a clean runtime error state: a non-sticky error left by an
    // earlier failed call (e.g. an allocation that ran out of memory) must not be reported
    // by this call's first cudaGetLastError. Sticky device faults persist regardless.
    (void)cudaGetLastError();
    static thread_local int ok_dev = -1;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "no CUDA device");
    if (dev == ok_dev) return DOTG_OK;
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return fail(DOTG_ECUDA, "dotg kernels are built for sm_100a; device is sm_" + std::to_string(major) +
                                    std::to_string(minor));
    ok_dev = dev;
    return DOTG_OK;
}

bool ranges_overlap(const void* x, size_t xb, const void* y, size_t yb) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(x), b0 = reinterpret_cast<uintptr_t>(y);
    return a0 < b0 + yb && b0 < a0 + xb;
}

// out may alias in exactly (same base, same extent); any other overlap is rejected.
bool bad_alias(const void* out, const void* in, size_t bytes) {
    return out != in && ranges_overlap(out, bytes, in, bytes);
}

int check_addsub(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m, size_t batch,
                 int layout) {
    if (layout != DOTG_ROW_MAJOR && layout != DOTG_INTERLEAVED) return fail(DOTG_EINVAL, "unknown layout");
    if (batch == 0) return DOTG_OK;
    if (m > 0 && (out == nullptr || a == nullptr || b == nullptr))
        return fail(DOTG_EINVAL, "dot add/sub: null operand");
    if (m > SIZE_MAX / 8 / batch) return fail(DOTG_EINVAL, "dot add/sub: size overflow");
    const size_t bytes = m * batch * sizeof(uint64_t);
    if (m > 0 && (bad_alias(out, a, bytes) || bad_alias(out, b, bytes)))
        return fail(DOTG_EINVAL, "dot add/sub: out may alias a or b only exactly (addsub.hpp:95-97)");
    if (flags != nullptr && m > 0 && ranges_overlap(flags, batch * 4, out, bytes))
        return fail(DOTG_EINVAL, "dot add/sub: flags overlap out");
    return DOTG_OK;
}

int check_mul(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch, int layout) {
    if (layout != DOTG_ROW_MAJOR && layout != DOTG_INTERLEAVED) return fail(DOTG_EINVAL, "unknown layout");
    if (m == 0) return fail(DOTG_EINVAL, "dot mul: operands need at least one limb");
    if (m > (size_t(1) << 24)) return fail(DOTG_EINVAL, "dot mul: limb count exceeds the column accumulator bound");
    if (batch == 0) return DOTG_OK;
    if (out == nullptr || a == nullptr || b == nullptr) return fail(DOTG_EINVAL, "dot mul: null operand");
    if (m > SIZE_MAX / 16 / batch) return fail(DOTG_EINVAL, "dot mul: size overflow");
    const size_t ib = m * batch * 8, ob = 2 * ib;
    if (ranges_overlap(out, ob, a, ib) || ranges_overlap(out, ob, b, ib))
        return fail(DOTG_EINVAL, "dot mul: out must not overlap the operands");
    return DOTG_OK;
}

int addsub_batch(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                 size_t batch, int layout, dotg_stream_t stream) {
    int rc = check_addsub(out, a, b, flags, m, batch, layout);
    if (rc != DOTG_OK) return rc;
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_addsub_batch(sub, out, a, b, flags, m, batch, layout,
                                              static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg add/sub batch launch");
}

int words(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, uint32_t* carry_out,
          dotg_stream_t stream) {
    int rc = check_addsub(out, a, b, nullptr, m, 1, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK) return rc;
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (m == 0) {
        if (carry_out == nullptr) return DOTG_OK;
        cudaError_t e = cudaMemsetAsync(carry_out, 0, sizeof(uint32_t), st);
        return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "memset");
    }
    const size_t sb = dotg::long_state_bytes(m);
    dotg::retain_stream_pool();
    void* scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, sb + 256, st);
    if (e != cudaSuccess) return fail(DOTG_ENOMEM, std::string("scratch: ") + cudaGetErrorString(e));
    uint32_t* agg = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) + sb);
    e = dotg::launch_long_local(sub, out, a, b, m, scratch, agg, st);
    if (e == cudaSuccess) e = dotg::launch_long_finish(sub, out, m, scratch, agg, 0, 1, carry_out, st);
    cudaError_t e2 = cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return cuda_fail(e, "dotg words launch");
    if (e2 != cudaSuccess) return cuda_fail(e2, "scratch free");
    return DOTG_OK;
}

// ---------------------------------------------------------------------------
// Host pipelines. One global staging context (host calls are synchronous). A call's
// work is cut into slices of ~24 MB of input, each H2D(a, b) -> kernel -> D2H(out,
// flags). Calls whose data fits kFlatMax get a device image of their own and run the
// flat pipeline (run_host_jobs_flat: uploads, kernels and downloads on three streams
// linked per slice by events); larger calls reuse kNS staging slots, slice k on stream
// k % kNS, so the H2D copy engine, the SMs and the D2H copy engine still work on three
// slices at once. Several jobs (e.g. a whole multi-size sweep) share one pipeline with no
// drain between jobs.
// ---------------------------------------------------------------------------
constexpr int kNS = 4;  // max pipeline depth; the used depth is host_streams()

// Tunables (environment, read once): DOTG_HOST_STREAMS (1..4, default 3) and
// DOTG_HOST_SLICE_MB (input MB per slice, default 24).
int host_streams() {
    static const int v = [] {
        const char* e = std::getenv("DOTG_HOST_STREAMS");
        const int x = e ? std::atoi(e) : 3;
        return x < 1 ? 1 : (x > kNS ? kNS : x);
    }();
    return v;
}
size_t slice_bytes() {
    static const size_t v = [] {
        const char* e = std::getenv("DOTG_HOST_SLICE_MB");
        const long x = e ? std::atol(e) : 24;
        return size_t(x < 1 ? 1 : x) << 20;
    }();
    return v;
}
// Multiply slices download as many bytes as they upload, so each slice's download is on
// the critical path once the uploads end: smaller slices shorten that drain, down to the
// size where per-copy and per-launch overhead takes over (tools/pcie_step_probe.py, 64 +
// 64 MB, download of chunk k after its upload: 2 MB 1.97 ms, 8 MB 1.57 ms, 24 MB 1.79 ms;
// the C3 / C4 host calls: 4 MB 1.22e8 / 2.99e7, 12 MB 1.44e8 / 3.59e7, 24 MB 1.39e8 /
// 3.48e7 pairs/s).
size_t mul_slice_bytes() {
    static const size_t v = [] {
        const char* e = std::getenv("DOTG_HOST_MUL_SLICE_MB");
        const long x = e ? std::atol(e) : 12;
        return size_t(x < 1 ? 1 : x) << 20;
    }();
    return v;
}

// Long-number host calls stream larger slices than batches (tools/c5_host_probe.py, 2^30
// limbs, pinned: 8 MB 62.6, 24 MB 64.3, 48 MB 74.1 GB/s vs 74.7 GB/s moving the same bytes
// with no kernels). DOTG_HOST_WORDS_SLICE_MB, input MB per slice (a and b), default 48.
size_t words_slice_bytes() {
    static const size_t v = [] {
        const char* e = std::getenv("DOTG_HOST_WORDS_SLICE_MB");
        const long x = e ? std::atol(e) : 48;
        return size_t(x < 1 ? 1 : x) << 20;
    }();
    return v;
}

struct HostCtx {
    std::mutex mu;
    int device = -1;
    cudaStream_t s[kNS] = {};
    char* buf[kNS] = {};
    size_t cap = 0;  // bytes per slot
    char* flat = nullptr;  // whole-call device image (flat pipeline)
    size_t flat_cap = 0;
    char* ring = nullptr;  // long-number slice ring (words_host)
    size_t ring_cap = 0;
    char* zc = nullptr;  // mapped pinned host staging for single short numbers (zero copy)
    char* zc_dev = nullptr;
    size_t zc_cap = 0;
    std::vector<cudaEvent_t> ev;
};
HostCtx g_host;

int host_prepare(size_t bytes_per_slot) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (g_host.device != dev) {
        for (int i = 0; i < kNS; ++i) {
            if (g_host.buf[i]) cudaFree(g_host.buf[i]);
            g_host.buf[i] = nullptr;
        }
        g_host.cap = 0;
        if (g_host.flat) cudaFree(g_host.flat);
        g_host.flat = nullptr;
        g_host.flat_cap = 0;
        if (g_host.ring) cudaFree(g_host.ring);
        g_host.ring = nullptr;
        g_host.ring_cap = 0;
        if (g_host.zc) cudaFreeHost(g_host.zc);
        g_host.zc = g_host.zc_dev = nullptr;
        g_host.zc_cap = 0;
        for (cudaEvent_t ev : g_host.ev) cudaEventDestroy(ev);
        g_host.ev.clear();  // events belong to the previous device
        for (int i = 0; i < kNS; ++i) {
            if ((e = cudaStreamCreateWithFlags(&g_host.s[i], cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_fail(e, "stream");
        }
        g_host.device = dev;
    }
    if (g_host.cap < bytes_per_slot) {
        for (int i = 0; i < kNS; ++i) {
            if (g_host.buf[i]) cudaFree(g_host.buf[i]);
            g_host.buf[i] = nullptr;
            if ((e = cudaMalloc(&g_host.buf[i], bytes_per_slot)) != cudaSuccess)
                return fail(DOTG_ENOMEM, std::string("staging: ") + cudaGetErrorString(e));
        }
        g_host.cap = bytes_per_slot;
    }
    return DOTG_OK;
}


size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct HostJob {  // op: 0 add, 1 sub, 2 mul; row-major host arrays
    int op;
    uint64_t* out;
    const uint64_t* a;
    const uint64_t* b;
    uint32_t* flags;
    size_t m, batch;
};

struct SliceGeom {
    size_t in_b, out_b, slice, sa, so, sf;
};

SliceGeom geom(const HostJob& j) {
    SliceGeom g{};
    g.in_b = j.m * 8;
    g.out_b = j.op == 2 ? 2 * j.m * 8 : j.m * 8;
    const size_t sb = j.op == 2 ? mul_slice_bytes() : slice_bytes();
    g.slice = std::min(std::max<size_t>(1, sb / (2 * g.in_b)), j.batch);
    g.sa = align_up(g.slice * g.in_b, 256);
    g.so = align_up(g.slice * g.out_b, 256);
    g.sf = align_up(g.slice * 4, 256);
    return g;
}

// Flat pipeline: the whole call's inputs and outputs get their own device image (no slot
// reuse), so the uploads run back to back on one stream, the kernels on a second and the
// downloads on a third, each slice linked only by its own two events: nothing ever waits
// for a download to free a staging slot. Used while the image fits in kFlatMax bytes.
constexpr size_t kFlatMax = size_t(16) << 30;
constexpr int kFlatNoMem = -1;  // run_host_jobs_flat: no room for the image, nothing enqueued

struct FlatGeom {
    size_t da, db, dout, dfl;  // offsets of the job's arrays in the image
};

size_t flat_layout(const HostJob* jobs, int n, std::vector<FlatGeom>& fg, size_t& slices) {
    size_t off = 0;
    slices = 0;
    fg.resize(size_t(n));
    for (int q = 0; q < n; ++q) {
        const HostJob& j = jobs[q];
        const SliceGeom g = geom(j);
        const size_t in = j.batch * g.in_b, outb = j.batch * g.out_b;
        fg[q].da = off;
        off += align_up(in, 256);
        fg[q].db = off;
        off += align_up(in, 256);
        fg[q].dout = off;
        off += align_up(outb, 256);
        fg[q].dfl = off;
        off += align_up(j.batch * 4, 256);
        slices += (j.batch + g.slice - 1) / g.slice;
    }
    return off;
}

int run_host_jobs_flat(const HostJob* jobs, int n, const std::vector<FlatGeom>& fg, size_t bytes, size_t slices) {
    cudaError_t e = cudaSuccess;
    if (g_host.flat_cap < bytes) {
        if (g_host.flat) cudaFree(g_host.flat);
        g_host.flat = nullptr;
        g_host.flat_cap = 0;
        if ((e = cudaMalloc(&g_host.flat, bytes)) != cudaSuccess) {
            g_host.flat = nullptr;
            cudaGetLastError();  // clear the (non-sticky) allocation error for the caller
            return kFlatNoMem;   // caller falls back to the staging-slot pipeline
        }
        g_host.flat_cap = bytes;
    }
    while (g_host.ev.size() < 2 * slices) {
        cudaEvent_t ev;
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "event");
        g_host.ev.push_back(ev);
    }
    cudaStream_t sh = g_host.s[0], sc = g_host.s[1], sd = g_host.s[2];
    size_t k = 0;
    for (int q = 0; q < n && e == cudaSuccess; ++q) {
        const HostJob& j = jobs[q];
        const SliceGeom g = geom(j);
        uint64_t* da = reinterpret_cast<uint64_t*>(g_host.flat + fg[q].da);
        uint64_t* db = reinterpret_cast<uint64_t*>(g_host.flat + fg[q].db);
        uint64_t* dout = reinterpret_cast<uint64_t*>(g_host.flat + fg[q].dout);
        uint32_t* dfl = reinterpret_cast<uint32_t*>(g_host.flat + fg[q].dfl);
        for (size_t p0 = 0; p0 < j.batch && e == cudaSuccess; p0 += g.slice, ++k) {
            const size_t cnt = std::min(g.slice, j.batch - p0);
            cudaEvent_t ev_in = g_host.ev[2 * k], ev_k = g_host.ev[2 * k + 1];
            e = cudaMemcpyAsync(da + p0 * j.m, j.a + p0 * j.m, cnt * g.in_b, cudaMemcpyHostToDevice, sh);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(db + p0 * j.m, j.b + p0 * j.m, cnt * g.in_b, cudaMemcpyHostToDevice, sh);
            if (e == cudaSuccess) e = cudaEventRecord(ev_in, sh);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(sc, ev_in, 0);
            if (e == cudaSuccess) {
                uint64_t* o = dout + p0 * (g.out_b / 8);
                e = j.op == 2 ? dotg::launch_mul_batch(o, da + p0 * j.m, db + p0 * j.m, j.m, cnt, 0, sc)
                              : dotg::launch_addsub_batch(j.op == 1, o, da + p0 * j.m, db + p0 * j.m,
                                                          j.flags ? dfl + p0 : nullptr, j.m, cnt, 0, sc);
            }
            if (e == cudaSuccess) e = cudaEventRecord(ev_k, sc);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, ev_k, 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(j.out + p0 * (g.out_b / 8), dout + p0 * (g.out_b / 8), cnt * g.out_b,
                                    cudaMemcpyDeviceToHost, sd);
            if (e == cudaSuccess && j.flags && j.op != 2)
                e = cudaMemcpyAsync(j.flags + p0, dfl + p0, cnt * 4, cudaMemcpyDeviceToHost, sd);
        }
    }
    cudaError_t es = cudaSuccess;
    for (cudaStream_t st : {sh, sc, sd}) {
        cudaError_t x = cudaStreamSynchronize(st);
        if (es == cudaSuccess) es = x;
    }
    if (g_host.flat_cap > (size_t(4) << 30)) {  // do not keep a huge image resident between calls
        cudaFree(g_host.flat);
        g_host.flat = nullptr;
        g_host.flat_cap = 0;
    }
    if (e != cudaSuccess) return cuda_fail(e, "dotg host pipeline");
    if (es != cudaSuccess) return cuda_fail(es, "dotg host pipeline sync");
    return DOTG_OK;
}

bool host_flat_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("DOTG_HOST_FLAT");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return v;
}

// Jobs must be validated; m > 0 and batch > 0 for every job.
int run_host_jobs(const HostJob* jobs, int n) {
    std::lock_guard<std::mutex> lk(g_host.mu);
    if (host_flat_enabled()) {
        std::vector<FlatGeom> fg;
        size_t slices = 0;
        const size_t bytes = flat_layout(jobs, n, fg, slices);
        if (bytes <= kFlatMax) {
            int rc = host_prepare(256);
            if (rc != DOTG_OK) return rc;
            rc = run_host_jobs_flat(jobs, n, fg, bytes, slices);
            if (rc != kFlatNoMem) return rc;
            // the image did not fit next to what the device already holds: the slot
            // pipeline below needs only kNS slices of staging
        }
    }
    size_t slot = 256;
    for (int q = 0; q < n; ++q) {
        const SliceGeom g = geom(jobs[q]);
        slot = std::max(slot, 2 * g.sa + g.so + g.sf);
    }
    int rc = host_prepare(slot);
    if (rc != DOTG_OK) return rc;
    cudaError_t e = cudaSuccess;
    size_t k = 0;
    for (int q = 0; q < n && e == cudaSuccess; ++q) {
        const HostJob& j = jobs[q];
        const SliceGeom g = geom(j);
        for (size_t p0 = 0; p0 < j.batch && e == cudaSuccess; p0 += g.slice, ++k) {
            const size_t cnt = std::min(g.slice, j.batch - p0);
            const int i = int(k % size_t(host_streams()));
            cudaStream_t st = g_host.s[i];
            uint64_t* da = reinterpret_cast<uint64_t*>(g_host.buf[i]);
            uint64_t* db = reinterpret_cast<uint64_t*>(g_host.buf[i] + g.sa);
            uint64_t* dout = reinterpret_cast<uint64_t*>(g_host.buf[i] + 2 * g.sa);
            uint32_t* dfl = reinterpret_cast<uint32_t*>(g_host.buf[i] + 2 * g.sa + g.so);
            // The previous use of this slot was enqueued on the same stream: ordered.
            e = cudaMemcpyAsync(da, j.a + p0 * j.m, cnt * g.in_b, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(db, j.b + p0 * j.m, cnt * g.in_b, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) {
                e = j.op == 2 ? dotg::launch_mul_batch(dout, da, db, j.m, cnt, 0, st)
                              : dotg::launch_addsub_batch(j.op == 1, dout, da, db, j.flags ? dfl : nullptr, j.m, cnt,
                                                          0, st);
            }
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(j.out + p0 * (g.out_b / 8), dout, cnt * g.out_b, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess && j.flags && j.op != 2)
                e = cudaMemcpyAsync(j.flags + p0, dfl, cnt * 4, cudaMemcpyDeviceToHost, st);
        }
    }
    cudaError_t es = cudaSuccess;
    for (int i = 0; i < kNS; ++i) {
        cudaError_t x = cudaStreamSynchronize(g_host.s[i]);
        if (es == cudaSuccess) es = x;
    }
    if (e != cudaSuccess) return cuda_fail(e, "dotg host pipeline");
    if (es != cudaSuccess) return cuda_fail(es, "dotg host pipeline sync");
    return DOTG_OK;
}

int batch_host(int op, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
               size_t batch) {
    int rc = op == 2 ? check_mul(out, a, b, m, batch, DOTG_ROW_MAJOR)
                     : check_addsub(out, a, b, flags, m, batch, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK) return rc;
    if (batch == 0) return DOTG_OK;
    if ((rc = check_device()) != DOTG_OK) return rc;
    if (op != 2 && m == 0) {
        if (flags) std::memset(flags, 0, batch * sizeof(uint32_t));
        return DOTG_OK;
    }
    const HostJob j{op, out, a, b, flags, m, batch};
    return run_host_jobs(&j, 1);
}

// Single long number from host spans through a RING of kRing device slots (a slice of a,
// b, out and its tile state each), never a whole device image: the number can exceed
// device memory, and nothing is mapped per call. Slices are independent shards
// (dotg_shard_*): uploads in order on one stream, the streaming pass of slice k on a second
// (as soon as its upload lands), and - because slice k's fix-up needs only the aggregates
// of slices 0..k, a carry scan ACROSS slices in slice order - its fix-up and download on a
// third right after its pass. The upload of slice k + kRing waits only for the download of
// slice k (same slot). H2D, kernels and D2H of different slices run concurrently.
constexpr int kRing = 6;
constexpr size_t kWordsSmall = size_t(1) << 16;  // limbs: below, one stream and the team kernel
constexpr size_t kWordsZeroCopy = 4096;           // limbs: below, mapped host memory, no copies
int words_host(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, uint32_t* carry) {
    int rc = check_addsub(out, a, b, nullptr, m, 1, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK) return rc;
    if (m == 0) {
        if (carry) *carry = 0;
        return DOTG_OK;
    }
    if ((rc = check_device()) != DOTG_OK) return rc;
    std::lock_guard<std::mutex> lk(g_host.mu);
    if ((rc = host_prepare(256)) != DOTG_OK) return rc;
    if (m <= kWordsZeroCopy) {
        // one short number (the reference's per-call use, e.g. Karatsuba's add_at): the
        // operands are copied by the CPU into mapped pinned memory and the team kernel
        // reads them and writes the result straight over PCIe - one launch and one
        // synchronisation, no copy-engine round trips (4096-bit add: ~36 -> ~10 us)
        const size_t ab = align_up(m * 8, 256);
        const size_t need = 3 * ab + 256;
        if (g_host.zc_cap < need) {
            if (g_host.zc) cudaFreeHost(g_host.zc);
            g_host.zc = g_host.zc_dev = nullptr;
            g_host.zc_cap = 0;
            const size_t cap = std::max<size_t>(need, size_t(1) << 20);
            void* hp = nullptr;
            cudaError_t ea = cudaHostAlloc(&hp, cap, cudaHostAllocMapped | cudaHostAllocPortable);
            void* dp = nullptr;
            if (ea == cudaSuccess) ea = cudaHostGetDevicePointer(&dp, hp, 0);
            if (ea != cudaSuccess) {
                if (hp) cudaFreeHost(hp);
                cudaGetLastError();
                return fail(DOTG_ENOMEM, std::string("words_host: ") + cudaGetErrorString(ea));
            }
            g_host.zc = static_cast<char*>(hp);
            g_host.zc_dev = static_cast<char*>(dp);
            g_host.zc_cap = cap;
        }
        std::memcpy(g_host.zc, a, m * 8);
        std::memcpy(g_host.zc + ab, b, m * 8);
        auto* za = reinterpret_cast<const uint64_t*>(g_host.zc_dev);
        auto* zb = reinterpret_cast<const uint64_t*>(g_host.zc_dev + ab);
        auto* zo = reinterpret_cast<uint64_t*>(g_host.zc_dev + 2 * ab);
        auto* zf = reinterpret_cast<uint32_t*>(g_host.zc_dev + 3 * ab);
        cudaStream_t s0 = g_host.s[0];
        cudaError_t e = dotg::launch_addsub_batch(sub, zo, za, zb, zf, m, 1, 0, s0);
        cudaError_t e2 = cudaStreamSynchronize(s0);
        if (e != cudaSuccess) return cuda_fail(e, "dotg words host");
        if (e2 != cudaSuccess) return cuda_fail(e2, "sync");
        std::memcpy(out, g_host.zc + 2 * ab, m * 8);
        if (carry) *carry = *reinterpret_cast<const uint32_t*>(g_host.zc + 3 * ab);
        return DOTG_OK;
    }
    if (m <= kWordsSmall) {
        // one short number: one stream, the batched team kernel with batch 1, one
        // synchronisation
        const size_t ab = align_up(m * 8, 256);
        if (g_host.ring_cap < 3 * ab + 256) {
            if (g_host.ring) cudaFree(g_host.ring);
            g_host.ring = nullptr;
            g_host.ring_cap = 0;
            cudaError_t ea = cudaMalloc(&g_host.ring, size_t(4) << 20);
            if (ea != cudaSuccess) {
                cudaGetLastError();
                return fail(DOTG_ENOMEM, std::string("words_host: ") + cudaGetErrorString(ea));
            }
            g_host.ring_cap = size_t(4) << 20;
        }
        uint64_t* da = reinterpret_cast<uint64_t*>(g_host.ring);
        uint64_t* db = reinterpret_cast<uint64_t*>(g_host.ring + ab);
        uint64_t* dout = reinterpret_cast<uint64_t*>(g_host.ring + 2 * ab);
        uint32_t* dfl = reinterpret_cast<uint32_t*>(g_host.ring + 3 * ab);
        cudaStream_t s0 = g_host.s[0];
        uint32_t hc = 0;
        cudaError_t e = cudaMemcpyAsync(da, a, m * 8, cudaMemcpyHostToDevice, s0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(db, b, m * 8, cudaMemcpyHostToDevice, s0);
        if (e == cudaSuccess) e = dotg::launch_addsub_batch(sub, dout, da, db, dfl, m, 1, 0, s0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, m * 8, cudaMemcpyDeviceToHost, s0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&hc, dfl, 4, cudaMemcpyDeviceToHost, s0);
        cudaError_t e2 = cudaStreamSynchronize(s0);
        if (e != cudaSuccess) return cuda_fail(e, "dotg words host");
        if (e2 != cudaSuccess) return cuda_fail(e2, "sync");
        if (carry) *carry = hc;
        return DOTG_OK;
    }
    const size_t slice = std::max<size_t>(4096, (words_slice_bytes() / 16) / 4096 * 4096);
    const size_t nsl = (m + slice - 1) / slice;
    const size_t sb = align_up(dotg::long_state_bytes(slice), 256);
    const size_t ab = align_up(slice * 8, 256);
    const size_t slot_bytes = 3 * ab + sb;
    const size_t ring_bytes = size_t(kRing) * slot_bytes + align_up(nsl * 8, 256) + 256;
    cudaError_t e = cudaSuccess;
    if (g_host.ring_cap < ring_bytes) {
        if (g_host.ring) cudaFree(g_host.ring);
        g_host.ring = nullptr;
        g_host.ring_cap = 0;
        if ((e = cudaMalloc(&g_host.ring, ring_bytes)) != cudaSuccess) {
            cudaGetLastError();
            return fail(DOTG_ENOMEM, std::string("words_host ring: ") + cudaGetErrorString(e));
        }
        g_host.ring_cap = ring_bytes;
    }
    char* base = g_host.ring;
    uint32_t* aggs = reinterpret_cast<uint32_t*>(base + size_t(kRing) * slot_bytes);
    uint32_t* dcarry = aggs + 2 * nsl;
    // events: [0, kRing) upload done per slot, [kRing, 2 kRing) pass done per slot,
    // [2 kRing, 3 kRing) download done per slot
    while (e == cudaSuccess && g_host.ev.size() < size_t(3 * kRing)) {
        cudaEvent_t ev;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) g_host.ev.push_back(ev);
    }
    cudaStream_t su = g_host.s[0], sk = g_host.s[1], sf = g_host.s[2];
    for (size_t k = 0; k < nsl && e == cudaSuccess; ++k) {
        const size_t l0 = k * slice, n = std::min(slice, m - l0);
        const int q = int(k % kRing);
        char* slot = base + size_t(q) * slot_bytes;
        uint64_t* da = reinterpret_cast<uint64_t*>(slot);
        uint64_t* db = reinterpret_cast<uint64_t*>(slot + ab);
        uint64_t* dout = reinterpret_cast<uint64_t*>(slot + 2 * ab);
        void* state = slot + 3 * ab;
        cudaEvent_t ev_up = g_host.ev[q], ev_pass = g_host.ev[kRing + q], ev_down = g_host.ev[2 * kRing + q];
        if (k >= size_t(kRing)) e = cudaStreamWaitEvent(su, ev_down, 0);  // slot free again
        if (e == cudaSuccess) e = cudaMemcpyAsync(da, a + l0, n * 8, cudaMemcpyHostToDevice, su);
        if (e == cudaSuccess) e = cudaMemcpyAsync(db, b + l0, n * 8, cudaMemcpyHostToDevice, su);
        if (e == cudaSuccess) e = cudaEventRecord(ev_up, su);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sk, ev_up, 0);
        if (e == cudaSuccess) e = dotg::launch_long_local(sub, dout, da, db, n, state, aggs + 2 * k, sk);
        if (e == cudaSuccess) e = cudaEventRecord(ev_pass, sk);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sf, ev_pass, 0);
        if (e == cudaSuccess)
            e = dotg::launch_long_finish(sub, dout, n, state, aggs, int(k), int(k + 1), k + 1 == nsl ? dcarry : nullptr,
                                         sf);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out + l0, dout, n * 8, cudaMemcpyDeviceToHost, sf);
        if (e == cudaSuccess) e = cudaEventRecord(ev_down, sf);
    }
    uint32_t hc = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hc, dcarry, 4, cudaMemcpyDeviceToHost, sf);
    cudaError_t e3 = cudaSuccess;
    for (cudaStream_t x : {su, sk, sf}) {
        cudaError_t y = cudaStreamSynchronize(x);
        if (e3 == cudaSuccess) e3 = y;
    }
    if (e != cudaSuccess) return cuda_fail(e, "dotg words host");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    if (carry) *carry = hc;
    return DOTG_OK;
}

}  // namespace

namespace dotg {
int api_fail(int code, const std::string& msg) { return fail(code, msg); }
int api_check_device() { return check_device(); }
int api_check_addsub_words(const uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m) {
    return check_addsub(const_cast<uint64_t*>(out), a, b, nullptr, m, 1, DOTG_ROW_MAJOR);
}
}  // namespace dotg

extern "C" {

int dotg_validate_width(int width) {
    if (width == 0 || width == 2 || width == 4 || width == 8) return DOTG_OK;
    return fail(DOTG_EINVAL, "unknown width selector");
}

const char* dotg_last_error(void) { return g_err.c_str(); }

const char* dotg_version(void) { return "dotg 0.1 sm_100a"; }

int dotg_device_sms(void) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return sms;
}

uint64_t dotg_kernel_launches(void) { return dotg::g_launches.load(); }

int dotg_set_mul_route(int route) {
    if (route != DOTG_MUL_AUTO && route != DOTG_MUL_IMAD && route != DOTG_MUL_IMMA)
        return -fail(DOTG_EINVAL, "set_mul_route: route must be DOTG_MUL_AUTO, DOTG_MUL_IMAD or DOTG_MUL_IMMA");
    return dotg::g_mul_route.exchange(route);
}

int dotg_fill_splitmix64(uint64_t* out, size_t n, uint64_t seed, uint64_t offset, dotg_stream_t stream) {
    if (n > 0 && out == nullptr) return fail(DOTG_EINVAL, "fill: null out");
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_fill_splitmix64(out, n, seed, offset, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "fill");
}

int dotg_add_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m, size_t batch,
                   int layout, dotg_stream_t stream) {
    return addsub_batch(false, out, a, b, flags, m, batch, layout, stream);
}

int dotg_sub_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m, size_t batch,
                   int layout, dotg_stream_t stream) {
    return addsub_batch(true, out, a, b, flags, m, batch, layout, stream);
}

int dotg_addsub_batch_strided(int sub, uint64_t* out, size_t ldo, const uint64_t* a, size_t lda, const uint64_t* b,
                              size_t ldb, uint32_t* flags, size_t m, size_t batch, dotg_stream_t stream) {
    if (batch == 0) return DOTG_OK;
    if (m > 0 && (out == nullptr || a == nullptr || b == nullptr))
        return fail(DOTG_EINVAL, "dot add/sub: null operand");
    if (batch > 1 && (ldo < m || lda < m || ldb < m))
        return fail(DOTG_EINVAL, "dot add/sub: row pitch below the limb count");
    const size_t mx = std::max(ldo, std::max(lda, ldb));
    if (m > 0 && (mx > SIZE_MAX / 8 / batch || m > SIZE_MAX / 8))
        return fail(DOTG_EINVAL, "dot add/sub: size overflow");
    // spanned bytes of each operand: (batch - 1) rows of pitch plus one row of m limbs
    auto span = [&](size_t ld) { return ((batch - 1) * ld + m) * sizeof(uint64_t); };
    if (m > 0) {
        const bool ea = out == a && ldo == lda, eb = out == b && ldo == ldb;
        if ((!ea && ranges_overlap(out, span(ldo), a, span(lda))) || (!eb && ranges_overlap(out, span(ldo), b, span(ldb))))
            return fail(DOTG_EINVAL, "dot add/sub: out may alias a or b only exactly (same pointer and pitch)");
        if (flags != nullptr && ranges_overlap(flags, batch * 4, out, span(ldo)))
            return fail(DOTG_EINVAL, "dot add/sub: flags overlap out");
    }
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    if (m == 0) {
        if (flags == nullptr) return DOTG_OK;
        cudaError_t e = cudaMemsetAsync(flags, 0, batch * sizeof(uint32_t), static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "memset");
    }
    cudaError_t e = dotg::launch_addsub_pitched(sub != 0, out, ldo, a, lda, b, ldb, flags, m, batch,
                                                static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg add/sub strided launch");
}

int dotg_mul_batch_strided(uint64_t* out, size_t ldo, const uint64_t* a, size_t lda, const uint64_t* b, size_t ldb,
                           size_t m, size_t batch, dotg_stream_t stream) {
    if (m == 0) return fail(DOTG_EINVAL, "dot mul: operands need at least one limb");
    if (m > (size_t(1) << 24)) return fail(DOTG_EINVAL, "dot mul: limb count exceeds the column accumulator bound");
    if (batch == 0) return DOTG_OK;
    if (out == nullptr || a == nullptr || b == nullptr) return fail(DOTG_EINVAL, "dot mul: null operand");
    if (batch > 1 && (lda < m || ldb < m || ldo < 2 * m))
        return fail(DOTG_EINVAL, "dot mul: row pitch below the limb count");
    const size_t mx = std::max(ldo, std::max(lda, ldb));
    if (mx > SIZE_MAX / 8 / batch) return fail(DOTG_EINVAL, "dot mul: size overflow");
    auto span = [&](size_t ld, size_t n) { return ((batch - 1) * ld + n) * sizeof(uint64_t); };
    if (ranges_overlap(out, span(ldo, 2 * m), a, span(lda, m)) || ranges_overlap(out, span(ldo, 2 * m), b, span(ldb, m)))
        return fail(DOTG_EINVAL, "dot mul: out must not overlap the operands");
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_mul_pitched(out, ldo, a, lda, b, ldb, m, batch, static_cast<cudaStream_t>(stream));
    if (e == cudaErrorMemoryAllocation) return fail(DOTG_ENOMEM, "dot mul: scratch allocation failed");
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg mul strided launch");
}

int dotg_addsub_grouped(const dotg_addsub_problem* problems, int n, dotg_stream_t stream) {
    if (n < 0 || (n > 0 && problems == nullptr)) return fail(DOTG_EINVAL, "grouped: bad problem list");
    if (n == 0) return DOTG_OK;
    std::vector<dotg::AddSubProblem> ps;
    std::vector<int> layouts;
    ps.reserve(size_t(n));
    for (int i = 0; i < n; ++i) {
        const dotg_addsub_problem& q = problems[i];
        if (q.op != 0 && q.op != 1) return fail(DOTG_EINVAL, "grouped: op must be 0 (add) or 1 (sub)");
        int rc = check_addsub(q.out, q.a, q.b, q.flags, q.m, q.batch, q.layout);
        if (rc != DOTG_OK) return rc;
        if (q.m > 0xffffffffull) return fail(DOTG_EINVAL, "grouped: m must fit 32 bits (use dotg_add_batch)");
        const size_t bytes = q.m * q.batch * 8;
        for (int j = 0; j < i && bytes; ++j) {
            const dotg_addsub_problem& o = problems[j];
            const size_t ob = o.m * o.batch * 8;
            if (!ob) continue;
            if (ranges_overlap(q.out, bytes, o.out, ob) || ranges_overlap(q.out, bytes, o.a, ob) ||
                ranges_overlap(q.out, bytes, o.b, ob) || ranges_overlap(o.out, ob, q.a, bytes) ||
                ranges_overlap(o.out, ob, q.b, bytes))
                return fail(DOTG_EINVAL, "grouped: problems must be independent (an output overlaps another problem)");
        }
        dotg::AddSubProblem P{};
        P.out = q.out;
        P.a = q.a;
        P.b = q.b;
        P.flags = q.flags;
        P.batch = q.batch;
        P.m = uint32_t(q.m);
        P.sub = uint32_t(q.op);
        ps.push_back(P);
        layouts.push_back(q.layout);
    }
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_addsub_group(ps.data(), layouts.data(), n, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg grouped launch");
}

int dotg_mul_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch, int layout,
                   dotg_stream_t stream) {
    int rc = check_mul(out, a, b, m, batch, layout);
    if (rc != DOTG_OK || batch == 0) return rc;
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_mul_batch(out, a, b, m, batch, layout, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg mul batch launch");
}

int dotg_mul52_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                     dotg_stream_t stream) {
    int rc = check_mul(out, a, b, m, batch, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK || batch == 0) return rc;
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_mul52_batch(out, a, b, m, batch, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg mul52 batch");
}

int dotg_mul52_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch) {
    int rc = check_mul(out, a, b, m, batch, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK || batch == 0) return rc;
    const uint64_t kHead = ~((uint64_t(1) << 52) - 1);
    for (size_t i = 0; i < m * batch; ++i)  // check_limbs (limbs.cpp:26-33)
        if ((a[i] | b[i]) & kHead)
            return fail(DOTG_EINVAL, "limb " + std::to_string(i % m) + " exceeds the configured limb width");
    if ((rc = check_device()) != DOTG_OK) return rc;
    std::lock_guard<std::mutex> lk(g_host.mu);
    if ((rc = host_prepare(256)) != DOTG_OK) return rc;
    cudaStream_t st = g_host.s[0];
    const size_t ib = align_up(m * batch * 8, 256);
    char* base = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), 4 * ib, st);
    if (e != cudaSuccess) return fail(DOTG_ENOMEM, std::string("mul52: ") + cudaGetErrorString(e));
    uint64_t* da = reinterpret_cast<uint64_t*>(base);
    uint64_t* db = reinterpret_cast<uint64_t*>(base + ib);
    uint64_t* dout = reinterpret_cast<uint64_t*>(base + 2 * ib);
    e = cudaMemcpyAsync(da, a, m * batch * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(db, b, m * batch * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = dotg::launch_mul52_batch(dout, da, db, m, batch, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, 2 * m * batch * 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaFreeAsync(base, st);
    cudaError_t e3 = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "dotg mul52");
    if (e2 != cudaSuccess) return cuda_fail(e2, "free");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    return DOTG_OK;
}

int dotg_karatsuba_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch, size_t theta,
                         dotg_stream_t stream) {
    if (theta < 1) return fail(DOTG_EINVAL, "karatsuba: threshold must be at least 1");  // mul.cpp:223-224
    int rc = check_mul(out, a, b, m, batch, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK || batch == 0) return rc;
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_karatsuba_batch(out, a, b, m, batch, theta, static_cast<cudaStream_t>(stream));
    if (e == cudaErrorMemoryAllocation) return fail(DOTG_ENOMEM, "karatsuba: scratch allocation failed");
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg karatsuba");
}

int dotg_karatsuba_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                              size_t theta) {
    if (theta < 1) return fail(DOTG_EINVAL, "karatsuba: threshold must be at least 1");
    int rc = check_mul(out, a, b, m, batch, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK || batch == 0) return rc;
    if ((rc = check_device()) != DOTG_OK) return rc;
    std::lock_guard<std::mutex> lk(g_host.mu);
    if ((rc = host_prepare(256)) != DOTG_OK) return rc;
    cudaStream_t st = g_host.s[0];
    const size_t ib = align_up(m * batch * 8, 256);
    char* base = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), 4 * ib, st);
    if (e != cudaSuccess) return fail(DOTG_ENOMEM, std::string("karatsuba: ") + cudaGetErrorString(e));
    uint64_t* da = reinterpret_cast<uint64_t*>(base);
    uint64_t* db = reinterpret_cast<uint64_t*>(base + ib);
    uint64_t* dout = reinterpret_cast<uint64_t*>(base + 2 * ib);
    e = cudaMemcpyAsync(da, a, m * batch * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(db, b, m * batch * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = dotg::launch_karatsuba_batch(dout, da, db, m, batch, theta, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, 2 * m * batch * 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaFreeAsync(base, st);
    cudaError_t e3 = cudaStreamSynchronize(st);
    if (e == cudaErrorMemoryAllocation) return fail(DOTG_ENOMEM, "karatsuba: scratch allocation failed");
    if (e != cudaSuccess) return cuda_fail(e, "dotg karatsuba host");
    if (e2 != cudaSuccess) return cuda_fail(e2, "free");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    return DOTG_OK;
}

int dotg_add_words(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, uint32_t* carry_out,
                   dotg_stream_t stream) {
    return words(false, out, a, b, m, carry_out, stream);
}

int dotg_sub_words(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, uint32_t* carry_out,
                   dotg_stream_t stream) {
    return words(true, out, a, b, m, carry_out, stream);
}

size_t dotg_shard_state_bytes(size_t m) { return dotg::long_state_bytes(m); }

int dotg_shard_local(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, void* state,
                     uint32_t* agg, dotg_stream_t stream) {
    int rc = check_addsub(out, a, b, nullptr, m, 1, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK) return rc;
    if (state == nullptr || agg == nullptr) return fail(DOTG_EINVAL, "shard: null state/agg");
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_long_local(sub != 0, out, a, b, m, state, agg, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg shard local");
}

int dotg_shard_finish(int sub, uint64_t* out, size_t m, void* state, const uint32_t* all_aggs, int rank, int world,
                      uint32_t* carry_out, dotg_stream_t stream) {
    if (world < 1 || rank < 0 || rank >= world) return fail(DOTG_EINVAL, "shard: bad rank/world");
    if (state == nullptr || all_aggs == nullptr) return fail(DOTG_EINVAL, "shard: null state/aggs");
    if (m > 0 && out == nullptr) return fail(DOTG_EINVAL, "shard: null out");
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_long_finish(sub != 0, out, m, state, all_aggs, rank, world, carry_out,
                                             static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "dotg shard finish");
}

int dotg_addsub_grouped_host(const dotg_addsub_problem* problems, int n) {
    if (n < 0 || (n > 0 && problems == nullptr)) return fail(DOTG_EINVAL, "grouped: bad problem list");
    std::vector<HostJob> jobs;
    for (int i = 0; i < n; ++i) {
        const dotg_addsub_problem& q = problems[i];
        if (q.op != 0 && q.op != 1) return fail(DOTG_EINVAL, "grouped: op must be 0 (add) or 1 (sub)");
        if (q.layout != DOTG_ROW_MAJOR) return fail(DOTG_EINVAL, "grouped host: row-major only");
        int rc = check_addsub(q.out, q.a, q.b, q.flags, q.m, q.batch, q.layout);
        if (rc != DOTG_OK) return rc;
        if (q.m > 0 && q.batch > 0) {
            // The pipeline uploads every problem's operands on one stream while results
            // download on another: a problem reading another's out (a chained problem) would
            // upload stale host data. Same independence rule as dotg_addsub_grouped.
            const size_t bytes = q.m * q.batch * 8;
            for (int j = 0; j < i; ++j) {
                const dotg_addsub_problem& o = problems[j];
                const size_t ob = o.m * o.batch * 8;
                if (!ob) continue;
                const bool clash = ranges_overlap(q.out, bytes, o.out, ob) || ranges_overlap(q.out, bytes, o.a, ob) ||
                                   ranges_overlap(q.out, bytes, o.b, ob) || ranges_overlap(o.out, ob, q.a, bytes) ||
                                   ranges_overlap(o.out, ob, q.b, bytes) ||
                                   (q.flags && (ranges_overlap(q.flags, q.batch * 4, o.out, ob) ||
                                                ranges_overlap(q.flags, q.batch * 4, o.a, ob) ||
                                                ranges_overlap(q.flags, q.batch * 4, o.b, ob) ||
                                                (o.flags && ranges_overlap(q.flags, q.batch * 4, o.flags, o.batch * 4)))) ||
                                   (o.flags && (ranges_overlap(o.flags, o.batch * 4, q.out, bytes) ||
                                                ranges_overlap(o.flags, o.batch * 4, q.a, bytes) ||
                                                ranges_overlap(o.flags, o.batch * 4, q.b, bytes)));
                if (clash)
                    return fail(DOTG_EINVAL,
                                "grouped host: problems must be independent (an output overlaps another problem)");
            }
        }
        if (q.batch == 0) continue;
        if (q.m == 0) {
            if (q.flags) std::memset(q.flags, 0, q.batch * sizeof(uint32_t));
            continue;
        }
        jobs.push_back(HostJob{q.op, q.out, q.a, q.b, q.flags, q.m, q.batch});
    }
    if (jobs.empty()) return DOTG_OK;
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    return run_host_jobs(jobs.data(), int(jobs.size()));
}

int dotg_addsub_stats(int sub, const uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                      int layout, int width, uint64_t* counters, dotg_stream_t stream) {
    int rc = dotg_validate_width(width);
    if (rc != DOTG_OK) return rc;
    if (layout != DOTG_ROW_MAJOR && layout != DOTG_INTERLEAVED) return fail(DOTG_EINVAL, "unknown layout");
    if (counters == nullptr) return fail(DOTG_EINVAL, "stats: null counters");
    if (m > 0 && batch > 0 && (out == nullptr || a == nullptr || b == nullptr))
        return fail(DOTG_EINVAL, "stats: null operand");
    if ((rc = check_device()) != DOTG_OK) return rc;
    const unsigned lanes = width == 0 ? 8u : unsigned(width);
    cudaError_t e = dotg::launch_addsub_stats(sub != 0, out, a, b, m, batch, layout, lanes, counters,
                                              static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "stats");
}

int dotg_addsub_phase_ticks(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                            size_t batch, uint64_t* ticks, dotg_stream_t stream) {
    int rc = check_addsub(out, a, b, flags, m, batch, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK) return rc;
    if (ticks == nullptr) return fail(DOTG_EINVAL, "phase ticks: null ticks");
    if (m == 0 || m > 256 || (m & (m - 1)) != 0)
        return fail(DOTG_ENOTSUP, "phase ticks: the timed kernel covers power-of-two m <= 256 (row-major)");
    if (batch == 0) return DOTG_OK;
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_addsub_timed(sub != 0, out, a, b, flags, m, batch, ticks,
                                              static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "phase ticks");
}

int dotg_addsub_phase_ticks_host(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                                 size_t m, size_t batch, uint64_t* ticks) {
    int rc = check_addsub(out, a, b, flags, m, batch, DOTG_ROW_MAJOR);
    if (rc != DOTG_OK) return rc;
    if (ticks == nullptr) return fail(DOTG_EINVAL, "phase ticks: null ticks");
    if (m == 0 || m > 256 || (m & (m - 1)) != 0)
        return fail(DOTG_ENOTSUP, "phase ticks: the timed kernel covers power-of-two m <= 256 (row-major)");
    if (batch == 0) return DOTG_OK;
    if ((rc = check_device()) != DOTG_OK) return rc;
    std::lock_guard<std::mutex> lk(g_host.mu);
    if ((rc = host_prepare(256)) != DOTG_OK) return rc;
    cudaStream_t st = g_host.s[0];
    const size_t ib = align_up(m * batch * 8, 256), fb = align_up(batch * 4, 256);
    char* base = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), 3 * ib + fb + 64, st);
    if (e != cudaSuccess) return fail(DOTG_ENOMEM, std::string("phase ticks: ") + cudaGetErrorString(e));
    uint64_t* da = reinterpret_cast<uint64_t*>(base);
    uint64_t* db = reinterpret_cast<uint64_t*>(base + ib);
    uint64_t* dout = reinterpret_cast<uint64_t*>(base + 2 * ib);
    uint32_t* dfl = reinterpret_cast<uint32_t*>(base + 3 * ib);
    uint64_t* dt = reinterpret_cast<uint64_t*>(base + 3 * ib + fb);
    e = cudaMemcpyAsync(da, a, m * batch * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(db, b, m * batch * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dt, ticks, 6 * 8, cudaMemcpyHostToDevice, st);  // accumulate
    if (e == cudaSuccess) e = dotg::launch_addsub_timed(sub != 0, dout, da, db, dfl, m, batch, dt, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, m * batch * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && flags) e = cudaMemcpyAsync(flags, dfl, batch * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ticks, dt, 6 * 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaFreeAsync(base, st);
    cudaError_t e3 = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "phase ticks host");
    if (e2 != cudaSuccess) return cuda_fail(e2, "free");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    return DOTG_OK;
}

int dotg_compare_batch(int32_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch, int layout,
                       dotg_stream_t stream) {
    if (layout != DOTG_ROW_MAJOR && layout != DOTG_INTERLEAVED) return fail(DOTG_EINVAL, "unknown layout");
    if (batch == 0) return DOTG_OK;
    if (out == nullptr || (m > 0 && (a == nullptr || b == nullptr))) return fail(DOTG_EINVAL, "compare: null operand");
    if (m > SIZE_MAX / 8 / batch) return fail(DOTG_EINVAL, "compare: size overflow");
    const size_t bytes = m * batch * 8;
    if (m > 0 && (ranges_overlap(out, batch * 4, a, bytes) || ranges_overlap(out, batch * 4, b, bytes)))
        return fail(DOTG_EINVAL, "compare: out overlaps an operand");
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_compare_batch(out, a, b, m, batch, layout, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "compare");
}

int dotg_chunk_batch(int sub, uint64_t* sums, uint32_t* carry_out, uint32_t* phase4_fired, const uint64_t* a,
                     const uint64_t* b, const uint32_t* carry_in, unsigned w, size_t batch, dotg_stream_t stream) {
    if (w < 1 || w > 8) return fail(DOTG_EINVAL, "chunk width must be in 1..8");  // addsub.cpp:174
    if (batch == 0) return DOTG_OK;
    if (sums == nullptr || carry_out == nullptr || a == nullptr || b == nullptr)
        return fail(DOTG_EINVAL, "chunk: null operand");
    if (batch > SIZE_MAX / 64) return fail(DOTG_EINVAL, "chunk: size overflow");
    const size_t bytes = batch * w * 8;
    if (bad_alias(sums, a, bytes) || bad_alias(sums, b, bytes))
        return fail(DOTG_EINVAL, "chunk: sums partially overlaps an operand");
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_chunk_batch(sub != 0, sums, carry_out, phase4_fired, a, b, carry_in, w, batch,
                                             static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "chunk");
}

int dotg_chunk_host(int sub, uint64_t* sums, uint32_t* carry_out, uint32_t* phase4_fired, const uint64_t* a,
                    const uint64_t* b, uint32_t carry_in, unsigned w) {
    if (w < 1 || w > 8) return fail(DOTG_EINVAL, "chunk width must be in 1..8");  // addsub.cpp:174
    if (carry_in > 1) return fail(DOTG_EINVAL, "carry_in must be 0 or 1");         // addsub.cpp:177
    if (sums == nullptr || carry_out == nullptr || a == nullptr || b == nullptr)
        return fail(DOTG_EINVAL, "chunk: null operand");
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    std::lock_guard<std::mutex> lk(g_host.mu);
    if ((rc = host_prepare(256)) != DOTG_OK) return rc;
    cudaStream_t st = g_host.s[0];
    // one staging block: a[8] b[8] sums[8] | carry_in carry_out fired
    uint64_t* d = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), 26 * 8, st);
    if (e != cudaSuccess) return fail(DOTG_ENOMEM, std::string("chunk: ") + cudaGetErrorString(e));
    uint32_t* flags = reinterpret_cast<uint32_t*>(d + 24);
    uint32_t res[2] = {0, 0};
    e = cudaMemcpyAsync(d, a, w * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d + 8, b, w * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(flags, &carry_in, 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = dotg::launch_chunk_batch(sub != 0, d + 16, flags + 1, flags + 2, d, d + 8, flags, w, 1, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sums, d + 16, w * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(res, flags + 1, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaFreeAsync(d, st);
    cudaError_t e3 = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "chunk host");
    if (e2 != cudaSuccess) return cuda_fail(e2, "free");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    *carry_out = res[0];
    if (phase4_fired != nullptr) *phase4_fired = res[1];
    return DOTG_OK;
}

}  // extern "C"

namespace {
int check_radix_bits(int k) {  // check_radix (limbs.cpp:21-24)
    return (k == 64 || k == 52) ? DOTG_OK : fail(DOTG_EINVAL, "RadixConfig: limb_bits must be 64 or 52");
}
int check_gather(size_t m) {  // gather_columns (mul.cpp:13-18)
    if (m == 0) return fail(DOTG_EINVAL, "dot mul: operands need at least one limb");
    if (m > (size_t(1) << 24)) return fail(DOTG_EINVAL, "dot mul: limb count exceeds the column accumulator bound");
    return DOTG_OK;
}

// Host form of one device stage: inputs copied in, outputs copied back, one sync.
struct HostBuf {
    void* host;
    size_t bytes;
    bool in, out;
};
template <typename F>
int run_staged(std::vector<HostBuf> bufs, const char* what, F&& fn) {
    int rc = check_device();
    if (rc != DOTG_OK) return rc;
    std::lock_guard<std::mutex> lk(g_host.mu);
    if ((rc = host_prepare(256)) != DOTG_OK) return rc;
    cudaStream_t st = g_host.s[0];
    size_t total = 0;
    std::vector<size_t> off;
    for (const HostBuf& b : bufs) {
        off.push_back(total);
        total += align_up(b.bytes, 256);
    }
    char* base = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), total ? total : 256, st);
    if (e != cudaSuccess) return fail(DOTG_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    std::vector<void*> dev;
    for (size_t i = 0; i < bufs.size(); ++i) {
        dev.push_back(base + off[i]);
        if (e == cudaSuccess && bufs[i].in && bufs[i].bytes)
            e = cudaMemcpyAsync(dev[i], bufs[i].host, bufs[i].bytes, cudaMemcpyHostToDevice, st);
    }
    if (e == cudaSuccess) e = fn(dev, st);
    for (size_t i = 0; i < bufs.size(); ++i)
        if (e == cudaSuccess && bufs[i].out && bufs[i].bytes)
            e = cudaMemcpyAsync(bufs[i].host, dev[i], bufs[i].bytes, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaFreeAsync(base, st);
    cudaError_t e3 = cudaStreamSynchronize(st);
    if (e == cudaErrorMemoryAllocation) return fail(DOTG_ENOMEM, std::string(what) + ": out of device memory");
    if (e != cudaSuccess) return cuda_fail(e, what);
    if (e2 != cudaSuccess) return cuda_fail(e2, "free");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    return DOTG_OK;
}
}  // namespace

extern "C" {

int dotg_gather_columns(uint64_t* m_a, uint64_t* m_b, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                        dotg_stream_t stream) {
    int rc = check_gather(m);
    if (rc != DOTG_OK || batch == 0) return rc;
    if (!m_a || !m_b || !a || !b) return fail(DOTG_EINVAL, "gather: null operand");
    if (batch > 65535) return fail(DOTG_EINVAL, "gather: at most 65535 operand pairs per call");
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_gather_columns(m_a, m_b, a, b, m, batch, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "gather");
}

int dotg_compute_partials(uint64_t* p_lo, uint64_t* p_hi, const uint64_t* m_a, const uint64_t* m_b, size_t n,
                          int limb_bits, dotg_stream_t stream) {
    int rc = check_radix_bits(limb_bits);
    if (rc != DOTG_OK || n == 0) return rc;
    if (!p_lo || !p_hi || !m_a || !m_b) return fail(DOTG_EINVAL, "partials: null operand");
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_partials(p_lo, p_hi, m_a, m_b, n, unsigned(limb_bits), static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "partials");
}

int dotg_align_and_reduce(uint64_t* columns, const uint64_t* p_lo, const uint64_t* p_hi, size_t m, size_t batch,
                          dotg_stream_t stream) {
    int rc = check_gather(m);
    if (rc != DOTG_OK || batch == 0) return rc;
    if (!columns || !p_lo || !p_hi) return fail(DOTG_EINVAL, "reduce: null operand");
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_align_reduce(columns, p_lo, p_hi, m, batch, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "reduce");
}

int dotg_carry_pass(uint64_t* out, uint32_t* out_limbs, size_t out_cap, const uint64_t* columns, size_t ncols,
                    size_t batch, int limb_bits, dotg_stream_t stream) {
    int rc = check_radix_bits(limb_bits);
    if (rc != DOTG_OK || batch == 0) return rc;
    if (out_cap < ncols + 2) return fail(DOTG_EINVAL, "carry pass: out_cap must be at least ncols + 2");
    if (!out || !out_limbs || (ncols > 0 && !columns)) return fail(DOTG_EINVAL, "carry pass: null operand");
    if ((rc = check_device()) != DOTG_OK) return rc;
    cudaError_t e = dotg::launch_carry_pass(out, out_limbs, out_cap, columns, ncols, batch, unsigned(limb_bits),
                                            static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DOTG_OK : cuda_fail(e, "carry pass");
}

int dotg_gather_columns_host(uint64_t* m_a, uint64_t* m_b, const uint64_t* a, const uint64_t* b, size_t m) {
    int rc = check_gather(m);
    if (rc != DOTG_OK) return rc;
    if (!m_a || !m_b || !a || !b) return fail(DOTG_EINVAL, "gather: null operand");
    if (m > (size_t(1) << 14)) return fail(DOTG_ENOMEM, "gather: m*m column buffers do not fit this call");
    const size_t ib = m * 8, ob = m * m * 8;
    return run_staged({{const_cast<uint64_t*>(a), ib, true, false}, {const_cast<uint64_t*>(b), ib, true, false},
                       {m_a, ob, false, true}, {m_b, ob, false, true}},
                      "gather", [&](std::vector<void*>& d, cudaStream_t st) {
                          return dotg::launch_gather_columns(static_cast<uint64_t*>(d[2]), static_cast<uint64_t*>(d[3]),
                                                             static_cast<uint64_t*>(d[0]),
                                                             static_cast<uint64_t*>(d[1]), m, 1, st);
                      });
}

int dotg_compute_partials_host(uint64_t* p_lo, uint64_t* p_hi, const uint64_t* m_a, const uint64_t* m_b, size_t n,
                               int limb_bits) {
    int rc = check_radix_bits(limb_bits);
    if (rc != DOTG_OK || n == 0) return rc;
    if (!p_lo || !p_hi || !m_a || !m_b) return fail(DOTG_EINVAL, "partials: null operand");
    const size_t nb = n * 8;
    return run_staged({{const_cast<uint64_t*>(m_a), nb, true, false}, {const_cast<uint64_t*>(m_b), nb, true, false},
                       {p_lo, nb, false, true}, {p_hi, nb, false, true}},
                      "partials", [&](std::vector<void*>& d, cudaStream_t st) {
                          return dotg::launch_partials(static_cast<uint64_t*>(d[2]), static_cast<uint64_t*>(d[3]),
                                                       static_cast<uint64_t*>(d[0]), static_cast<uint64_t*>(d[1]), n,
                                                       unsigned(limb_bits), st);
                      });
}

int dotg_align_and_reduce_host(uint64_t* columns, const uint64_t* p_lo, const uint64_t* p_hi, size_t m) {
    int rc = check_gather(m);
    if (rc != DOTG_OK) return rc;
    if (!columns || !p_lo || !p_hi) return fail(DOTG_EINVAL, "reduce: null operand");
    if (m > (size_t(1) << 14)) return fail(DOTG_ENOMEM, "reduce: m*m partial buffers do not fit this call");
    const size_t pb = m * m * 8, cb = 2 * m * 16;
    return run_staged({{const_cast<uint64_t*>(p_lo), pb, true, false}, {const_cast<uint64_t*>(p_hi), pb, true, false},
                       {columns, cb, false, true}},
                      "reduce", [&](std::vector<void*>& d, cudaStream_t st) {
                          return dotg::launch_align_reduce(static_cast<uint64_t*>(d[2]), static_cast<uint64_t*>(d[0]),
                                                           static_cast<uint64_t*>(d[1]), m, 1, st);
                      });
}

int dotg_compare_host(int32_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch) {
    if (batch == 0) return DOTG_OK;
    if (out == nullptr || (m > 0 && (a == nullptr || b == nullptr))) return fail(DOTG_EINVAL, "compare: null operand");
    if (m > SIZE_MAX / 8 / batch) return fail(DOTG_EINVAL, "compare: size overflow");
    const size_t ib = m * batch * 8;
    return run_staged({{const_cast<uint64_t*>(a), ib, true, false}, {const_cast<uint64_t*>(b), ib, true, false},
                       {out, batch * 4, false, true}},
                      "compare", [&](std::vector<void*>& d, cudaStream_t st) {
                          return dotg::launch_compare_batch(static_cast<int32_t*>(d[2]),
                                                            static_cast<uint64_t*>(d[0]),
                                                            static_cast<uint64_t*>(d[1]), m, batch, 0, st);
                      });
}

int dotg_carry_census(unsigned k, uint64_t* counts) {
    if (k < 1 || k > 16) return fail(DOTG_EINVAL, "carry_census: k must be in 1..16");  // oracle.cpp:66
    if (counts == nullptr) return fail(DOTG_EINVAL, "carry_census: null output");
    return run_staged({{counts, 16, false, true}}, "carry census", [&](std::vector<void*>& d, cudaStream_t st) {
        return dotg::launch_carry_census(k, static_cast<uint64_t*>(d[0]), st);
    });
}

int dotg_mc_carry(uint64_t samples, uint64_t seed, uint64_t* carries) {
    if (carries == nullptr) return fail(DOTG_EINVAL, "mc carry: null output");
    return run_staged({{carries, 8, false, true}}, "mc carry", [&](std::vector<void*>& d, cudaStream_t st) {
        return dotg::launch_mc_carry(samples, seed, static_cast<uint64_t*>(d[0]), st);
    });
}

int dotg_carry_pass_host(uint64_t* out, uint32_t* out_limbs, size_t out_cap, const uint64_t* columns, size_t ncols,
                         int limb_bits) {
    int rc = check_radix_bits(limb_bits);
    if (rc != DOTG_OK) return rc;
    if (out_cap < ncols + 2) return fail(DOTG_EINVAL, "carry pass: out_cap must be at least ncols + 2");
    if (!out || !out_limbs || (ncols > 0 && !columns)) return fail(DOTG_EINVAL, "carry pass: null operand");
    return run_staged({{const_cast<uint64_t*>(columns), ncols * 16, true, false}, {out, out_cap * 8, false, true},
                       {out_limbs, 4, false, true}},
                      "carry pass", [&](std::vector<void*>& d, cudaStream_t st) {
                          return dotg::launch_carry_pass(static_cast<uint64_t*>(d[1]), static_cast<uint32_t*>(d[2]),
                                                         out_cap, static_cast<uint64_t*>(d[0]), ncols, 1,
                                                         unsigned(limb_bits), st);
                      });
}

int dotg_words_host_stats(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, int width,
                          uint32_t* carry, uint64_t* chunks, uint64_t* fires) {
    int rc = dotg_validate_width(width);
    if (rc != DOTG_OK) return rc;
    if ((rc = check_addsub(out, a, b, nullptr, m, 1, DOTG_ROW_MAJOR)) != DOTG_OK) return rc;
    if (m == 0) {
        if (carry) *carry = 0;
        return DOTG_OK;
    }
    if ((rc = check_device()) != DOTG_OK) return rc;
    std::lock_guard<std::mutex> lk(g_host.mu);
    if ((rc = host_prepare(256)) != DOTG_OK) return rc;
    cudaStream_t st = g_host.s[0];
    const size_t ab = align_up(m * 8, 256);
    const size_t sb = align_up(dotg::long_state_bytes(m), 256);
    char* base = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), 3 * ab + sb + 256, st);
    if (e != cudaSuccess) return fail(DOTG_ENOMEM, std::string("stats: ") + cudaGetErrorString(e));
    uint64_t* da = reinterpret_cast<uint64_t*>(base);
    uint64_t* db = reinterpret_cast<uint64_t*>(base + ab);
    uint64_t* dout = reinterpret_cast<uint64_t*>(base + 2 * ab);
    char* state = base + 3 * ab;
    uint32_t* agg = reinterpret_cast<uint32_t*>(state + sb);  // agg[0..1], carry agg[2]
    uint64_t* cnt = reinterpret_cast<uint64_t*>(state + sb + 64);
    uint64_t hc[2] = {0, 0};
    uint32_t hcarry = 0;
    e = cudaMemcpyAsync(da, a, m * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(db, b, m * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, 16, st);
    if (e == cudaSuccess) e = dotg::launch_long_local(sub != 0, dout, da, db, m, state, agg, st);
    if (e == cudaSuccess) e = dotg::launch_long_finish(sub != 0, dout, m, state, agg, 0, 1, agg + 2, st);
    if (e == cudaSuccess)
        e = dotg::launch_addsub_stats(sub != 0, dout, da, db, m, 1, DOTG_ROW_MAJOR, width == 0 ? 8u : unsigned(width),
                                      cnt, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, m * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hcarry, agg + 2, 4, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaFreeAsync(base, st);
    cudaError_t e3 = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "stats words");
    if (e2 != cudaSuccess) return cuda_fail(e2, "free");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    if (carry) *carry = hcarry;
    if (chunks) *chunks += hc[0];
    if (fires) *fires += hc[1];
    return DOTG_OK;
}

int dotg_add_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                        size_t batch) {
    return batch_host(0, out, a, b, flags, m, batch);
}
int dotg_sub_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                        size_t batch) {
    return batch_host(1, out, a, b, flags, m, batch);
}
int dotg_mul_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch) {
    return batch_host(2, out, a, b, nullptr, m, batch);
}
int dotg_add_words_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, uint32_t* carry) {
    return words_host(false, out, a, b, m, carry);
}
int dotg_sub_words_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, uint32_t* carry) {
    return words_host(true, out, a, b, m, carry);
}

}  // extern "C"
