// C-ABI implementation (include/visrt.h): scene lifecycle, matrix calls.
// Never throws across the boundary; errors land in a thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <mutex>

#include "capi_internal.h"
#include "device.h"
#include "host_geom.h"

namespace visrt {
struct PairArgs;
cudaError_t launch_pair_bits(const PairArgs& a, int device, cudaStream_t st);
cudaError_t launch_pair_detail(const PairArgs& a, int device, cudaStream_t st);
cudaError_t launch_prefilter(const DevScene& s, long long npairs, long long* d_sel, long long* d_count,
                             void*& temp, size_t& temp_bytes, cudaStream_t st);
cudaError_t launch_split_pairs(const long long* sel, long long m, int n, int32_t* ci, int32_t* cj,
                               cudaStream_t st);
cudaError_t launch_clear_pairs(unsigned long long* bits, int words, const int32_t* ci, const int32_t* cj,
                               long long m, cudaStream_t st);
}  // namespace visrt


namespace {

thread_local std::string g_err;

using visrt::ck;
using visrt::CudaError;
using visrt::UsageError;
using visrt::VisError;

template <class F>
int guarded(F&& f) {
    return visrt::capi_guard(std::forward<F>(f));
}

template <class T>
T* dev_upload(const std::vector<T>& v, std::vector<void*>& allocs) {
    T* p = nullptr;
    const size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
    ck(cudaMalloc(&p, bytes), "cudaMalloc");
    allocs.push_back(p);
    if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    return p;
}

template <class T>
T* dev_alloc(size_t count, std::vector<void*>& allocs) {
    return visrt::dalloc<T>(count, allocs);
}

// Scene state lives in ONE device arena from the device's stream-ordered
// memory pool (kept resident: release threshold = max), filled by ONE copy
// from a process-wide pinned staging buffer — scene creation/destruction stay
// at O(10 us) of driver work instead of ~20 cudaMalloc/cudaFree/pageable
// copies (the e2e path creates a scene per step).
struct Arena {
    struct Part {
        const void* src;
        size_t bytes, off;
    };
    std::vector<Part> parts;
    size_t total = 0;
    size_t add(const void* src, size_t bytes) {
        const size_t off = total;
        parts.push_back({src, bytes, off});
        total += (std::max<size_t>(bytes, 16) + 255) & ~size_t(255);
        return off;
    }
};

std::mutex g_stage_mu;
void* g_stage = nullptr;
size_t g_stage_bytes = 0;

void pool_setup(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done.push_back(device);
}

}  // namespace

struct visrt_scene {
    visrt::HostScene hs;
    visrt::DevScene ds;
    int device = 0;
    std::vector<void*> allocs;
    void* arena = nullptr;   // pooled device arena holding every scene array
    visrt::ChainCache chain_cache;
    int64_t upload_bytes = 0;
    unsigned long long* d_bits = nullptr;
    unsigned long long* d_counter = nullptr;
    long long* d_count = nullptr;
    // candidate state (PREFILTERED)
    long long* d_sel = nullptr;
    long long sel_cap = 0;
    int32_t* d_ci = nullptr;
    int32_t* d_cj = nullptr;
    uint8_t* d_cbit = nullptr;
    long long ncand = 0;
    std::vector<int32_t> ci, cj;
    std::vector<uint8_t> cbit;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    ~visrt_scene() {
        if (device < 0) return;   // host-only handle
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        for (void* p : allocs) visrt::BlockCache::get().release(p);
        if (arena) {
            cudaFreeAsync(arena, 0);
            cudaStreamSynchronize(0);
        }
        if (d_sel) cudaFree(d_sel);
        if (d_ci) cudaFree(d_ci);
        if (d_cj) cudaFree(d_cj);
        if (d_cbit) cudaFree(d_cbit);
        if (temp) cudaFree(temp);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        cudaSetDevice(cur);
    }

    void ensure_cand(long long m) {
        if (m <= sel_cap) return;
        if (d_sel) cudaFree(d_sel);
        if (d_ci) cudaFree(d_ci);
        if (d_cj) cudaFree(d_cj);
        if (d_cbit) cudaFree(d_cbit);
        ck(cudaMalloc(&d_sel, std::max<long long>(m, 1) * sizeof(long long)), "cudaMalloc sel");
        ck(cudaMalloc(&d_ci, std::max<long long>(m, 1) * sizeof(int32_t)), "cudaMalloc ci");
        ck(cudaMalloc(&d_cj, std::max<long long>(m, 1) * sizeof(int32_t)), "cudaMalloc cj");
        ck(cudaMalloc(&d_cbit, std::max<long long>(m, 1)), "cudaMalloc cbit");
        sel_cap = m;
    }
};

namespace visrt {
void set_last_error(const std::string& msg) { g_err = msg; }
ChainCache& scene_chain_cache(visrt_scene* s) { return s->chain_cache; }
const DevScene& scene_dev(const visrt_scene* s) { return s->ds; }
const HostScene& scene_host(const visrt_scene* s) { return s->hs; }
int scene_device(const visrt_scene* s) { return s->device; }
}  // namespace visrt

namespace {

visrt::PairArgs base_args(visrt_scene* sc) {
    visrt::PairArgs a{};
    a.s = sc->ds;
    a.bits = sc->d_bits;
    a.counter = sc->d_counter;
    return a;
}

double tests_alg_all(const visrt::HostScene& hs) {
    // Σ_{i<j} S(i,j) (N-2), grouped by (nv, ns) class.
    std::vector<std::pair<std::pair<int, int>, long long>> cls;
    for (int i = 0; i < hs.n; ++i) {
        const auto key = std::make_pair(hs.nv[i], hs.ns[i]);
        auto it = std::find_if(cls.begin(), cls.end(), [&](const auto& c) { return c.first == key; });
        if (it == cls.end()) cls.push_back({key, 1});
        else ++it->second;
    }
    double total = 0.0;
    for (size_t a = 0; a < cls.size(); ++a) {
        for (size_t b = a; b < cls.size(); ++b) {
            const double S = visrt::sightline_count(cls[a].first.first, cls[a].first.second,
                                                    cls[b].first.first, cls[b].first.second);
            const double cnt = a == b ? 0.5 * cls[a].second * (cls[a].second - 1)
                                      : static_cast<double>(cls[a].second) * cls[b].second;
            total += S * cnt;
        }
    }
    return total * (hs.n - 2);
}

}  // namespace

extern "C" {

const char* visrt_last_error(void) { return g_err.c_str(); }
int visrt_version(void) { return 1; }

int visrt_scene_create(const visrt_facets_v1* f, int device, visrt_scene** out) {
    return guarded([&] {
        if (!f || !out) throw UsageError("null argument");
        *out = nullptr;
        auto sc = std::make_unique<visrt_scene>();
        sc->device = device;
        visrt::ingest(*f, sc->hs);
        if (device < 0) {   // host-only handle: ingest products, no device state
            sc->ds.n = sc->hs.n;
            *out = sc.release();
            return;
        }
        ck(cudaSetDevice(device), "cudaSetDevice");
        const auto& hs = sc->hs;
        auto& ds = sc->ds;
        ds.n = hs.n;
        ds.maxv = hs.maxv;
        ds.words = (hs.n + 63) / 64;
        Arena ar;
        auto add = [&](const auto& v) { return ar.add(v.data(), v.size() * sizeof(v[0])); };
        ds.rec_stride = hs.maxv <= 4 ? visrt::RecLayout<4>::kStride : visrt::RecLayout<8>::kStride;
        // device copies: the sweeps read the occluder records and culling boxes
        // in Morton order (srec / sbox); the tree's unfolding reads the records
        // by face index (rec: no inv[] indirection on its dependent chain)
        const auto& rec = hs.maxv <= 4 ? hs.rec4 : hs.rec8;
        // (first vertex, normal) per face, 48 B dense: the image tree's plane
        // tests gather it per candidate (one sector pair instead of two lines)
        std::vector<double> pn(static_cast<size_t>(hs.n) * 6);
        for (int f = 0; f < hs.n; ++f)
            for (int d = 0; d < 3; ++d) {
                pn[6 * static_cast<size_t>(f) + d] = hs.pts[static_cast<size_t>(f) * VISRT_MAX_VERTS * 3 + d];
                pn[6 * static_cast<size_t>(f) + 3 + d] = hs.normal[3 * static_cast<size_t>(f) + d];
            }
        const size_t o_pn = add(pn);
        const size_t o_rec = add(rec), o_samples = add(hs.samples), o_pts = add(hs.pts), o_normal = add(hs.normal),
                     o_seg = add(hs.seg), o_aabb = add(hs.aabb), o_nv = add(hs.nv), o_ns = add(hs.ns),
                     o_orient = add(hs.orient), o_seg_ok = add(hs.seg_ok), o_sbox = add(hs.sbox),
                     o_tbox = add(hs.tbox), o_gbox = add(hs.gbox), o_cbox = add(hs.cbox), o_srec = add(hs.srec), o_perm = add(hs.perm), o_inv = add(hs.inv),
                     o_tframe = add(hs.tframe), o_qbox = add(hs.qbox);
        const size_t data_bytes = ar.total;   // the scene data; the buffers below are device-only
        const size_t o_bits = ar.add(nullptr, static_cast<size_t>(hs.n) * ds.words * 8);
        const size_t o_counter = ar.add(nullptr, 4 * 8);
        const size_t o_count = ar.add(nullptr, 2 * 8);
        pool_setup(device);
        ck(cudaMallocAsync(&sc->arena, ar.total, 0), "cudaMallocAsync arena");
        {
            std::lock_guard<std::mutex> lk(g_stage_mu);
            if (g_stage_bytes < ar.total) {
                if (g_stage) cudaFreeHost(g_stage);
                g_stage = nullptr;
                g_stage_bytes = 0;
                ck(cudaHostAlloc(&g_stage, ar.total, cudaHostAllocDefault), "cudaHostAlloc staging");
                g_stage_bytes = ar.total;
            }
            char* st = static_cast<char*>(g_stage);
            for (const auto& pt : ar.parts)
                if (pt.src && pt.bytes) std::memcpy(st + pt.off, pt.src, pt.bytes);
            ck(cudaMemcpyAsync(sc->arena, g_stage, data_bytes, cudaMemcpyHostToDevice, 0), "H2D scene");
            ck(cudaStreamSynchronize(0), "sync");
        }
        char* base = static_cast<char*>(sc->arena);
        auto at = [&](size_t off) { return static_cast<void*>(base + off); };
        ds.rec = static_cast<const double*>(at(o_rec));
        ds.samples = static_cast<const double*>(at(o_samples));
        ds.pts = static_cast<const double*>(at(o_pts));
        ds.normal = static_cast<const double*>(at(o_normal));
        ds.pn = static_cast<const double*>(at(o_pn));
        ds.seg = static_cast<const double*>(at(o_seg));
        ds.aabb = static_cast<const double*>(at(o_aabb));
        ds.nv = static_cast<const int32_t*>(at(o_nv));
        ds.ns = static_cast<const int32_t*>(at(o_ns));
        ds.orient = static_cast<const int32_t*>(at(o_orient));
        ds.seg_ok = static_cast<const int32_t*>(at(o_seg_ok));
        ds.box = nullptr;
        ds.sbox = static_cast<const float*>(at(o_sbox));
        ds.tbox = static_cast<const float*>(at(o_tbox));
        ds.gbox = static_cast<const float*>(at(o_gbox));
        ds.cbox = static_cast<const float*>(at(o_cbox));
        ds.srec = static_cast<const double*>(at(o_srec));
        ds.tframe = static_cast<const float*>(at(o_tframe));
        ds.qbox = static_cast<const uint32_t*>(at(o_qbox));
        ds.perm = static_cast<const int32_t*>(at(o_perm));
        ds.inv = static_cast<const int32_t*>(at(o_inv));
        sc->d_bits = static_cast<unsigned long long*>(at(o_bits));
        sc->d_counter = static_cast<unsigned long long*>(at(o_counter));
        sc->d_count = static_cast<long long*>(at(o_count));
        ds.ntiles = hs.ntiles;
        ds.nchunks = hs.nchunks;
        ds.ngroups = hs.ngroups;
        sc->upload_bytes = static_cast<int64_t>(data_bytes);   // the one H2D copy of the scene
        ds.ox = hs.origin[0];
        ds.oy = hs.origin[1];
        ds.oz = hs.origin[2];
        ck(cudaEventCreate(&sc->ev0), "event");
        ck(cudaEventCreate(&sc->ev1), "event");
        *out = sc.release();
    });
}

void visrt_scene_destroy(visrt_scene* s) { delete s; }

int visrt_scene_nfaces(const visrt_scene* s) { return s ? s->hs.n : 0; }

int64_t visrt_scene_upload_bytes(const visrt_scene* s) { return s ? s->upload_bytes : 0; }

int visrt_scene_ingest(const visrt_scene* s, double* normal, int32_t* orientation, double* seg,
                       int32_t* seg_ok) {
    return guarded([&] {
        if (!s) throw UsageError("null scene");
        const auto& hs = s->hs;
        if (normal) std::memcpy(normal, hs.normal.data(), hs.normal.size() * sizeof(double));
        if (orientation) std::memcpy(orientation, hs.orient.data(), hs.orient.size() * sizeof(int32_t));
        if (seg) std::memcpy(seg, hs.seg.data(), hs.seg.size() * sizeof(double));
        if (seg_ok) std::memcpy(seg_ok, hs.seg_ok.data(), hs.seg_ok.size() * sizeof(int32_t));
    });
}

const uint64_t* visrt_matrix_bits_device(const visrt_scene* s) {
    return s ? reinterpret_cast<const uint64_t*>(s->d_bits) : nullptr;
}

// Pairs (i, j), i < j, of rows [row0, row1) and their S(i,j)(N-2) reference tests.
static void row_block_work(const visrt::HostScene& hs, int row0, int row1, long long& pairs, double& tests) {
    const int n = hs.n;
    pairs = 0;
    double t = 0.0;
    // count of faces per (nv, ns) class among j > i, swept from the last row up
    std::vector<std::pair<std::pair<int, int>, long long>> cls;
    for (int i = n - 1; i >= row0; --i) {
        if (i < row1) {
            for (const auto& c : cls)
                t += static_cast<double>(visrt::sightline_count(hs.nv[i], hs.ns[i], c.first.first, c.first.second)) *
                     c.second;
            pairs += n - 1 - i;
        }
        const auto key = std::make_pair(hs.nv[i], hs.ns[i]);
        auto it = std::find_if(cls.begin(), cls.end(), [&](const auto& c) { return c.first == key; });
        if (it == cls.end()) cls.push_back({key, 1});
        else ++it->second;
    }
    tests = t * (n - 2);
}

static int pair_visibility_impl(visrt_scene* sc, uint32_t flags, int32_t row0, int32_t row1, uint64_t* bits_host,
                                visrt_stats* stats, void* stream);

int visrt_pair_visibility(visrt_scene* sc, uint32_t flags, uint64_t* bits_host, visrt_stats* stats,
                          void* stream) {
    return pair_visibility_impl(sc, flags, 0, 0, bits_host, stats, stream);
}

int visrt_pair_visibility_rows(visrt_scene* sc, uint32_t flags, int32_t row0, int32_t row1, uint64_t* bits_host,
                               visrt_stats* stats, void* stream) {
    const int n = sc ? sc->hs.n : 0;
    if (sc && (row0 < 0 || row1 > n || row0 >= row1))
        return guarded([&] { throw UsageError("row block must satisfy 0 <= row0 < row1 <= nfaces"); });
    if (sc && (flags & VISRT_PAIRS_PREFILTERED))
        return guarded([&] { throw UsageError("row blocks shard the all-pairs (B) matrix only"); });
    return pair_visibility_impl(sc, flags, row0, row1, bits_host, stats, stream);
}

static int pair_visibility_impl(visrt_scene* sc, uint32_t flags, int32_t row0, int32_t row1, uint64_t* bits_host,
                                visrt_stats* stats, void* stream) {
    return guarded([&] {
        if (!sc) throw UsageError("null scene");
        const bool pref = (flags & VISRT_PAIRS_PREFILTERED) != 0;
        if (!pref && !(flags & VISRT_PAIRS_ALL)) throw UsageError("flags must select ALL or PREFILTERED");
        visrt::ScopedDevice dev_guard(sc);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int n = sc->hs.n;
        const long long npairs = static_cast<long long>(n) * (n - 1) / 2;
        const size_t bit_words = static_cast<size_t>(n) * sc->ds.words;
        // The selected count bounds every later buffer; size for the worst case
        // once per scene, before the timed region (allocation is not build work).
        if (pref) sc->ensure_cand(npairs);
        ck(cudaEventRecord(sc->ev0, st), "event");
        ck(cudaMemsetAsync(sc->d_bits, 0, bit_words * 8, st), "memset bits");
        ck(cudaMemsetAsync(sc->d_counter, 0, 4 * sizeof(unsigned long long), st), "memset counter");
        visrt::PairArgs a = base_args(sc);
        long long ncand = npairs;
        if (pref) {
            ck(visrt::launch_prefilter(sc->ds, npairs, sc->d_sel, sc->d_count, sc->temp, sc->temp_bytes, st),
               "prefilter");
            ck(cudaMemcpyAsync(&ncand, sc->d_count, sizeof(long long), cudaMemcpyDeviceToHost, st), "D2H count");
            ck(cudaStreamSynchronize(st), "sync");
            ck(visrt::launch_split_pairs(sc->d_sel, ncand, n, sc->d_ci, sc->d_cj, st), "split");
            a.npairs = ncand;
            a.ci = sc->d_ci;
            a.cj = sc->d_cj;
            a.cbit = sc->d_cbit;
        } else {
            a.npairs = npairs;
            if (row1) {   // a row block: absolute pair indices [pbegin, npairs)
                auto before = [n](long long r) { return r * (2LL * n - r - 1) / 2; };   // pairs in rows < r
                a.row0 = row0;
                a.row1 = row1;
                a.pbegin = before(row0);
                a.npairs = before(row1);
            }
        }
        if (a.npairs - a.pbegin > 0) ck(visrt::launch_pair_bits(a, sc->device, st), "k_pair_bits");
        ck(cudaEventRecord(sc->ev1, st), "event");
        unsigned long long counters[4] = {0, 0, 0, 0};
        ck(cudaMemcpyAsync(counters, sc->d_counter, sizeof(counters), cudaMemcpyDeviceToHost, st), "D2H ctr");
        if (pref) {
            sc->ncand = ncand;
            sc->ci.resize(ncand);
            sc->cj.resize(ncand);
            sc->cbit.resize(ncand);
            if (ncand > 0) {
                ck(cudaMemcpyAsync(sc->ci.data(), sc->d_ci, ncand * 4, cudaMemcpyDeviceToHost, st), "D2H ci");
                ck(cudaMemcpyAsync(sc->cj.data(), sc->d_cj, ncand * 4, cudaMemcpyDeviceToHost, st), "D2H cj");
                ck(cudaMemcpyAsync(sc->cbit.data(), sc->d_cbit, ncand, cudaMemcpyDeviceToHost, st), "D2H cbit");
            }
        }
        ck(cudaStreamSynchronize(st), "sync");
        long long admitted = 0;
        if (pref) {
            // pair_admitted also drops pairs whose bouncing range degenerates in
            // some plane (src/vismatrix.cpp:622-624): host angle records.
            std::vector<int32_t> drop_i, drop_j;
            for (long long k = 0; k < ncand; ++k) {
                if (!sc->cbit[k]) continue;
                if (visrt::pair_range_degenerate(sc->hs, sc->ci[k], sc->cj[k])) {
                    sc->cbit[k] = 0;
                    drop_i.push_back(sc->ci[k]);
                    drop_j.push_back(sc->cj[k]);
                } else {
                    ++admitted;
                }
            }
            if (!drop_i.empty()) {
                // the selection buffer (npairs x 8 B, consumed by the split
                // above) holds the drop lists: no allocation, and the copies
                // are ordered on the caller's stream before the clear kernel
                int32_t* di = reinterpret_cast<int32_t*>(sc->d_sel);
                int32_t* dj = di + drop_i.size();
                ck(cudaMemcpyAsync(di, drop_i.data(), drop_i.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
                ck(cudaMemcpyAsync(dj, drop_j.data(), drop_j.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
                ck(visrt::launch_clear_pairs(sc->d_bits, sc->ds.words, di, dj,
                                             static_cast<long long>(drop_i.size()), st), "clear");
                ck(cudaStreamSynchronize(st), "sync");
            }
        }
        if (bits_host) {
            ck(cudaMemcpyAsync(bits_host, sc->d_bits, bit_words * 8, cudaMemcpyDeviceToHost, st), "D2H bits");
            ck(cudaStreamSynchronize(st), "sync");
        }
        if (stats) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, sc->ev0, sc->ev1);
            stats->pairs = npairs;
            stats->candidates = ncand;
            stats->tests_exec = static_cast<int64_t>(counters[1]);
            stats->sweeps = static_cast<int64_t>(counters[2]);
            stats->tiles = static_cast<int64_t>(counters[3]);
            stats->ms = ms;
            if (pref) {
                double t = 0.0;
                for (long long k = 0; k < ncand; ++k) {
                    const int i = sc->ci[k], j = sc->cj[k];
                    t += visrt::sightline_count(sc->hs.nv[i], sc->hs.ns[i], sc->hs.nv[j], sc->hs.ns[j]);
                }
                stats->tests_alg = t * (n - 2);
                stats->admitted = admitted;
            } else if (row1) {
                long long bp = 0;
                row_block_work(sc->hs, row0, row1, bp, stats->tests_alg);
                stats->pairs = bp;
                stats->candidates = bp;
                stats->admitted = -1;
            } else {
                stats->tests_alg = tests_alg_all(sc->hs);
                stats->admitted = -1;
            }
        }
    });
}

int64_t visrt_candidates(const visrt_scene* sc, int32_t* ci, int32_t* cj, uint8_t* admitted) {
    if (!sc) return -1;
    if (ci) std::memcpy(ci, sc->ci.data(), sc->ci.size() * 4);
    if (cj) std::memcpy(cj, sc->cj.data(), sc->cj.size() * 4);
    if (admitted) std::memcpy(admitted, sc->cbit.data(), sc->cbit.size());
    return sc->ncand;
}

int visrt_pair_detail(visrt_scene* sc, int64_t npairs, const int32_t* ci, const int32_t* cj, int8_t* kind,
                      int64_t* blk_off, int32_t* blk_idx, int64_t blk_cap, visrt_stats* stats, void* stream) {
    return guarded([&] {
        if (!sc) throw UsageError("null scene");
        visrt::ScopedDevice dev_guard(sc);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int n = sc->hs.n;
        for (int64_t k = 0; k < npairs; ++k) {
            if (ci[k] < 0 || ci[k] >= n || cj[k] < 0 || cj[k] >= n)
                throw UsageError("face index out of range");
            if (ci[k] == cj[k]) throw VisError("occlusion judgment needs two distinct faces");
        }
        const int words32 = (n + 31) / 32;
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        int32_t* d_ci = dev_alloc<int32_t>(npairs, tmp);
        int32_t* d_cj = dev_alloc<int32_t>(npairs, tmp);
        int8_t* d_kind = dev_alloc<int8_t>(npairs, tmp);
        uint32_t* d_mask = dev_alloc<uint32_t>(static_cast<size_t>(npairs) * words32, tmp);
        ck(cudaMemcpyAsync(d_ci, ci, npairs * 4, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(d_cj, cj, npairs * 4, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemsetAsync(d_mask, 0, static_cast<size_t>(npairs) * words32 * 4, st), "memset");
        ck(cudaMemsetAsync(sc->d_counter, 0, 4 * sizeof(unsigned long long), st), "memset");
        ck(cudaEventRecord(sc->ev0, st), "event");
        visrt::PairArgs a = base_args(sc);
        a.npairs = npairs;
        a.ci = d_ci;
        a.cj = d_cj;
        a.kind = d_kind;
        a.blk_mask = d_mask;
        a.blk_words = words32;
        if (npairs > 0) ck(visrt::launch_pair_detail(a, sc->device, st), "k_pair_detail");
        ck(cudaEventRecord(sc->ev1, st), "event");
        std::vector<uint32_t> mask(static_cast<size_t>(npairs) * words32);
        unsigned long long counters[2] = {0, 0};
        if (npairs > 0) {
            ck(cudaMemcpyAsync(kind, d_kind, npairs, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(mask.data(), d_mask, mask.size() * 4, cudaMemcpyDeviceToHost, st), "D2H");
        }
        ck(cudaMemcpyAsync(counters, sc->d_counter, sizeof(counters), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        int64_t off = 0;
        for (int64_t k = 0; k < npairs; ++k) {
            if (blk_off) blk_off[k] = off;
            for (int w = 0; w < words32; ++w) {
                uint32_t m = mask[static_cast<size_t>(k) * words32 + w];
                while (m) {
                    const int b = __builtin_ctz(m);
                    m &= m - 1;
                    if (blk_idx && off < blk_cap) blk_idx[off] = w * 32 + b;
                    ++off;
                }
            }
        }
        if (blk_off) blk_off[npairs] = off;
        if (blk_idx && off > blk_cap) throw UsageError("blocker capacity too small");
        if (stats) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, sc->ev0, sc->ev1);
            double t = 0.0;
            for (int64_t k = 0; k < npairs; ++k)
                t += visrt::sightline_count(sc->hs.nv[ci[k]], sc->hs.ns[ci[k]], sc->hs.nv[cj[k]], sc->hs.ns[cj[k]]);
            stats->pairs = npairs;
            stats->candidates = npairs;
            stats->admitted = -1;
            stats->tests_alg = t * (n - 2);
            stats->tests_exec = static_cast<int64_t>(counters[1]);
            stats->ms = ms;
        }
    });
}

}  // extern "C"

// --- entry points implemented in later milestones (regions.cu / tree.cu) ---
