// Binary matrix / pair-graph cache: the on-disk
// hand-off between a preprocessing run and later query runs, replacing the
// reference's text format "visrt-matrix v1" (src/vismatrix.cpp:805-968), which
// stores every InterVisEntry as text and cannot hold config-4 scale.
//
// Content: the admitted order-1 bit matrix (pair_admitted, N x ceil(N/64)
// uint64, symmetric) and the feasible order-2 triples (p, t, a) — everything
// else in an InterVisMatrix (records, criteria, subranges, blockers, images,
// orders >= 3 by Markov-2 growth) is re-derived from these two by the same
// code that built it (rt::build_matrix), so the cache is exact and small:
// config 4's 22k facets need 61 MB of bits (+ 12 B per triple) instead of
// ~1 KB of text per entry.
//
// Layout (little endian):
//   char[8]  "VISRTMB1"
//   u32 version (1), u32 flags (bit 0: triples present)
//   i32 nfaces, i32 max_order
//   u64 scene fingerprint (FNV-1a over face vertex counts + coordinates)
//   i64 ntriples
//   u64 bits[nfaces * ceil(nfaces/64)]
//   i32 triples[3 * ntriples]
//   u64 payload checksum (FNV-1a over bits + triples)
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "capi_internal.h"

namespace visrt {
namespace {

constexpr char kMagic[8] = {'V', 'I', 'S', 'R', 'T', 'M', 'B', '1'};

struct Fnv {
    uint64_t h = 1469598103934665603ull;
    void add(const void* p, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        for (size_t k = 0; k < n; ++k) {
            h ^= b[k];
            h *= 1099511628211ull;
        }
    }
};

uint64_t scene_fingerprint(const HostScene& hs) {
    Fnv f;
    f.add(&hs.n, sizeof(hs.n));
    for (int i = 0; i < hs.n; ++i) {
        f.add(&hs.nv[i], sizeof(int32_t));
        f.add(&hs.pts[static_cast<size_t>(i) * VISRT_MAX_VERTS * 3], sizeof(double) * 3 * hs.nv[i]);
    }
    return f.h;
}

struct Header {
    char magic[8];
    uint32_t version, flags;
    int32_t n, max_order;
    uint64_t fingerprint;
    int64_t ntriples;
};

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

}  // namespace
}  // namespace visrt

extern "C" int visrt_cache_save(const char* path, const visrt_scene* sc, int32_t max_order, const uint64_t* bits,
                                int64_t ntriples, const int32_t* triples) {
    return visrt::capi_guard([&] {
        if (!path || !sc || !bits) throw visrt::UsageError("null argument");
        if (ntriples < 0 || (ntriples > 0 && !triples)) throw visrt::UsageError("bad triple list");
        const visrt::HostScene& hs = visrt::scene_host(sc);
        const size_t nw = static_cast<size_t>(hs.n) * ((hs.n + 63) / 64);
        visrt::Header h{};
        std::memcpy(h.magic, visrt::kMagic, 8);
        h.version = 1;
        h.flags = ntriples > 0 ? 1u : 0u;
        h.n = hs.n;
        h.max_order = max_order;
        h.fingerprint = visrt::scene_fingerprint(hs);
        h.ntriples = ntriples;
        visrt::File fp;
        fp.f = std::fopen(path, "wb");
        if (!fp.f) throw visrt::VisError(std::string("cannot write matrix cache '") + path + "'");
        visrt::Fnv ck;
        ck.add(bits, nw * 8);
        if (ntriples) ck.add(triples, static_cast<size_t>(ntriples) * 12);
        bool ok = std::fwrite(&h, sizeof(h), 1, fp.f) == 1 && std::fwrite(bits, 8, nw, fp.f) == nw;
        if (ok && ntriples) ok = std::fwrite(triples, 12, static_cast<size_t>(ntriples), fp.f) == static_cast<size_t>(ntriples);
        if (ok) ok = std::fwrite(&ck.h, 8, 1, fp.f) == 1;
        if (!ok) throw visrt::VisError(std::string("short write on matrix cache '") + path + "'");
    });
}

// triples == NULL: header only (max_order, ntriples); bits may be NULL too.
extern "C" int visrt_cache_load(const char* path, const visrt_scene* sc, int32_t* max_order, uint64_t* bits,
                                int32_t* triples, int64_t cap, int64_t* ntriples) {
    return visrt::capi_guard([&] {
        if (!path || !sc) throw visrt::UsageError("null argument");
        const visrt::HostScene& hs = visrt::scene_host(sc);
        visrt::File fp;
        fp.f = std::fopen(path, "rb");
        if (!fp.f) throw visrt::VisError(std::string("cannot open matrix cache '") + path + "'");
        visrt::Header h{};
        if (std::fread(&h, sizeof(h), 1, fp.f) != 1 || std::memcmp(h.magic, visrt::kMagic, 8) != 0 || h.version != 1)
            throw visrt::VisError(std::string("matrix cache '") + path + "' has an unknown header");
        if (h.n != hs.n || h.fingerprint != visrt::scene_fingerprint(hs))
            throw std::runtime_error("matrix cache '" + std::string(path) + "' was built for a different scene");
        if (max_order) *max_order = h.max_order;
        if (ntriples) *ntriples = h.ntriples;
        if (!bits && !triples) return;
        if (triples && cap < h.ntriples) throw visrt::UsageError("triple capacity below the cached count");
        const size_t nw = static_cast<size_t>(h.n) * ((h.n + 63) / 64);
        std::vector<uint64_t> b(nw);
        std::vector<int32_t> t(static_cast<size_t>(h.ntriples) * 3);
        uint64_t stored = 0;
        bool ok = std::fread(b.data(), 8, nw, fp.f) == nw;
        if (ok && h.ntriples) ok = std::fread(t.data(), 12, static_cast<size_t>(h.ntriples), fp.f) == static_cast<size_t>(h.ntriples);
        if (ok) ok = std::fread(&stored, 8, 1, fp.f) == 1;
        visrt::Fnv ck;
        ck.add(b.data(), nw * 8);
        if (h.ntriples) ck.add(t.data(), t.size() * 4);
        if (!ok || ck.h != stored) throw visrt::VisError(std::string("matrix cache '") + path + "' is truncated or corrupt");
        if (bits) std::memcpy(bits, b.data(), nw * 8);
        if (triples && !t.empty()) std::memcpy(triples, t.data(), t.size() * 4);
    });
}
