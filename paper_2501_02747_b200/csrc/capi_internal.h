// Helpers shared by the C-ABI translation units (never exposed in visrt.h).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
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

template <class T>
T* dalloc(size_t count, std::vector<void*>& allocs) {
    T* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(count * sizeof(T), 16)), "cudaMalloc");
    allocs.push_back(p);
    return p;
}

struct FreeGuard {
    std::vector<void*>& v;
    ~FreeGuard() {
        for (void* p : v) cudaFree(p);
    }
};

}  // namespace visrt
