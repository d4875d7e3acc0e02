// Helpers shared by the C-ABI translation units (never exposed in visrt.h).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "device.h"

namespace visrt {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct VisError : std::runtime_error {        // reference VisibilityError
    using std::runtime_error::runtime_error;
};
struct PlaceError : std::runtime_error {      // reference PlacementError
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Run f(); map exceptions to visrt.h status codes (never throws).
template <class F>
int capi_guard(F&& f) {
    try {
        f();
        return VISRT_OK;
    } catch (const CudaError& e) {
        set_last_error(e.what());
        return VISRT_E_CUDA;
    } catch (const UsageError& e) {
        set_last_error(e.what());
        return VISRT_E_USAGE;
    } catch (const VisError& e) {
        set_last_error(e.what());
        return VISRT_E_VISIBILITY;
    } catch (const PlaceError& e) {
        set_last_error(e.what());
        return VISRT_E_PLACEMENT;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return VISRT_E_SCENE;
    }
}

// Result cache of visrt_chain_triples (the two-call sizing pattern would
// otherwise run the kernel twice): keyed by a hash of the admitted bits.
struct ChainCache {
    bool valid = false;
    uint64_t key = 0;
    std::vector<int32_t> tri;   // sorted (p, t, a)
    int64_t pairs = 0, candidates = 0;
    float ms = 0.f;
};
ChainCache& scene_chain_cache(visrt_scene* s);

const DevScene& scene_dev(const visrt_scene* s);
const HostScene& scene_host(const visrt_scene* s);
int scene_device(const visrt_scene* s);

struct ScopedDevice {
    explicit ScopedDevice(const visrt_scene* s) {
        if (!s) throw UsageError("null scene");
        if (scene_device(s) < 0) throw UsageError("host-only scene handle (device < 0) has no device state");
        ck(cudaSetDevice(scene_device(s)), "cudaSetDevice");
    }
};

// Caching allocator for the per-call scratch buffers (power-of-two buckets
// per device, blocks returned by FreeGuard are reused, never released): every
// C-ABI call synchronises its stream before returning, so a returned block is
// idle. Repeated calls (trajectory bisection rounds, e2e steps) then pay no
// cudaMalloc/cudaFree. Blocks above 1 GiB bypass the cache.
struct BlockCache {
    std::mutex mu;
    std::map<std::pair<int, size_t>, std::vector<void*>> free_blocks;
    std::map<void*, std::pair<int, size_t>> owner;
    static BlockCache& get() {
        static BlockCache c;
        return c;
    }
    static size_t bucket(size_t bytes) {
        size_t b = 256;
        while (b < bytes) b <<= 1;
        return b;
    }
    void* alloc(size_t bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (bytes > (size_t(1) << 30)) {
            void* p = nullptr;
            ck(cudaMalloc(&p, bytes), "cudaMalloc");
            return p;
        }
        const size_t b = bucket(bytes);
        {
            std::lock_guard<std::mutex> lk(mu);
            auto& fl = free_blocks[{dev, b}];
            if (!fl.empty()) {
                void* p = fl.back();
                fl.pop_back();
                return p;
            }
        }
        void* p = nullptr;
        ck(cudaMalloc(&p, b), "cudaMalloc");
        std::lock_guard<std::mutex> lk(mu);
        owner[p] = {dev, b};
        return p;
    }
    void release(void* p) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = owner.find(p);
        if (it == owner.end()) {
            cudaFree(p);   // uncached (large) block
            return;
        }
        free_blocks[it->second].push_back(p);
    }
};

template <class T>
T* dalloc(size_t count, std::vector<void*>& allocs) {
    T* p = static_cast<T*>(BlockCache::get().alloc(std::max<size_t>(count * sizeof(T), 16)));
    allocs.push_back(p);
    return p;
}

struct FreeGuard {
    std::vector<void*>& v;
    ~FreeGuard() {
        for (void* p : v) BlockCache::get().release(p);
    }
};

}  // namespace visrt
