// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI adapter around the UNMODIFIED reference implementation compiled from
// /root/reference/proj/src/*.cpp with -Drt=visrt_ref (recipe: oracle/Makefile,
// output: oracle/_ref/libvisrt_ref.so). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.
//
// The BASELINE configs are open boxes on a tiled ground, which the reference's
// Scene::finalize rejects (closed shells only, one ground face:
// proj/src/scene.cpp:126-143, proj/include/rt/scene.hpp:77). The facet-soup
// adapter below fills Scene's private face index directly:
// face_ptrs_/face_index_ exactly as register_face does (proj/src/scene.cpp:86-97)
// and Face::orientation exactly as classify_orientation (proj/src/scene.cpp:19-24).
// Every hot-path function then runs unchanged (they only use scene.faces(),
// scene.face(id|idx) and scene.edges()). Consequences: no edges (no diffraction,
// empty AngleRecord::edge_id) and inside_building() is always false.

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#define private public
#include "rt/scene.hpp"
#undef private
#include "rt/geom.hpp"
#include "rt/raytracer.hpp"
#include "rt/vismatrix.hpp"
#include "rt/vistable.hpp"
#include "rt/em.hpp"

#include "ref_capi.h"

namespace R = visrt_ref;

namespace {

thread_local std::string g_err;

struct RefScene {
    R::Scene scene;
    std::vector<R::Face> soup;  // storage for facet-soup faces (stable addresses)
};

// proj/src/scene.cpp:19-24 (anonymous namespace there, restated verbatim in behaviour)
R::Orientation classify(const R::Vec3& n) {
    const double ax = std::abs(n.x), ay = std::abs(n.y), az = std::abs(n.z);
    if (ax <= R::kEpsAng && ay <= R::kEpsAng) return R::Orientation::Horizontal;
    if (az <= R::kEpsAng) return R::Orientation::Vertical;
    return R::Orientation::Oblique;
}

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

int error_code(const std::exception& e) {
    if (dynamic_cast<const R::VisibilityError*>(&e)) return 1;
    if (dynamic_cast<const R::PlacementError*>(&e)) return 2;
    if (dynamic_cast<const R::SceneError*>(&e)) return 3;
    return 5;
}

}  // namespace

extern "C" {

const char* vref_last_error(void) { return g_err.c_str(); }

// Facet soup: nfaces rings; ids is a '\0'-separated concatenation of ids.
void* vref_scene_from_soup(int32_t nfaces, const int32_t* vert_off, const double* verts,
                           const char* ids) {
    try {
        auto* rs = new RefScene();
        rs->soup.reserve(static_cast<size_t>(nfaces));
        const char* idp = ids;
        for (int32_t i = 0; i < nfaces; ++i) {
            R::Face f;
            f.id = idp;
            idp += f.id.size() + 1;
            f.material = "concrete";
            std::vector<R::Vec3> pts;
            for (int32_t k = vert_off[i]; k < vert_off[i + 1]; ++k) {
                pts.push_back({verts[3 * k], verts[3 * k + 1], verts[3 * k + 2]});
            }
            f.poly = R::ConvexPolygon::from_points(std::move(pts));
            f.orientation = classify(f.poly.normal);
            f.index = i;
            rs->soup.push_back(std::move(f));
        }
        rs->scene.materials.push_back({"concrete", 5.31, 0.139});
        for (int32_t i = 0; i < nfaces; ++i) {
            rs->scene.face_ptrs_.push_back(&rs->soup[static_cast<size_t>(i)]);
            rs->scene.face_index_[rs->soup[static_cast<size_t>(i)].id] = i;
        }
        return rs;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Closed-shell scene through the reference's own Scene::finalize: faces with
// building index b >= 0 go to buildings[b] (ids '\0'-separated), the one face
// with b < 0 (if any) is the ground.
void* vref_scene_from_shells(int32_t nfaces, const int32_t* vert_off, const double* verts, const char* ids,
                             const int32_t* building, int32_t nbuildings, const char* building_ids) {
    try {
        auto* rs = new RefScene();
        rs->scene.materials.push_back({"concrete", 5.31, 0.139});
        const char* bp = building_ids;
        for (int32_t b = 0; b < nbuildings; ++b) {
            R::Building bd;
            bd.id = bp;
            bp += bd.id.size() + 1;
            rs->scene.buildings.push_back(std::move(bd));
        }
        const char* idp = ids;
        for (int32_t i = 0; i < nfaces; ++i) {
            R::Face f;
            f.id = idp;
            idp += f.id.size() + 1;
            f.material = "concrete";
            std::vector<R::Vec3> pts;
            for (int32_t k = vert_off[i]; k < vert_off[i + 1]; ++k)
                pts.push_back({verts[3 * k], verts[3 * k + 1], verts[3 * k + 2]});
            f.poly = R::ConvexPolygon::from_points(std::move(pts));
            if (building[i] >= 0) rs->scene.buildings[static_cast<size_t>(building[i])].faces.push_back(std::move(f));
            else rs->scene.ground = std::move(f);
        }
        rs->scene.finalize();
        return rs;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Reference loader (closed-shell fixture scenes; only usable where the JSON exists).
void* vref_scene_load(const char* path) {
    try {
        // Scene holds raw Face pointers into itself (proj/include/rt/scene.hpp:97):
        // construct it in place from the prvalue, never move-assign it.
        return new RefScene{R::load_scene(path), {}};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void vref_scene_free(void* h) { delete static_cast<RefScene*>(h); }

// save_scene (proj/src/scene.cpp:327-375) of a loaded scene; 0 ok, -1 error.
int32_t vref_scene_save(void* h, const char* path) {
    try {
        R::save_scene(static_cast<RefScene*>(h)->scene, path);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int32_t vref_nfaces(void* h) {
    return static_cast<int32_t>(static_cast<RefScene*>(h)->scene.faces().size());
}

int32_t vref_nedges(void* h) {
    return static_cast<int32_t>(static_cast<RefScene*>(h)->scene.edges().size());
}

// Face export: id, label xy/vert, building id, vertex ring, orientation.
int32_t vref_face_export(void* h, int32_t idx, char* id, int32_t idcap, char* bld, int32_t bldcap,
                         char* lab_xy, char* lab_vert, int32_t labcap, double* pts, int32_t ptcap,
                         double* normal) {
    const R::Face& f = static_cast<RefScene*>(h)->scene.face(idx);
    std::snprintf(id, static_cast<size_t>(idcap), "%s", f.id.c_str());
    std::snprintf(bld, static_cast<size_t>(bldcap), "%s", f.building.c_str());
    std::snprintf(lab_xy, static_cast<size_t>(labcap), "%s", f.labels.xy.c_str());
    std::snprintf(lab_vert, static_cast<size_t>(labcap), "%s", f.labels.vert.c_str());
    const int32_t n = static_cast<int32_t>(f.poly.pts.size());
    for (int32_t k = 0; k < n && k < ptcap; ++k) {
        pts[3 * k] = f.poly.pts[k].x;
        pts[3 * k + 1] = f.poly.pts[k].y;
        pts[3 * k + 2] = f.poly.pts[k].z;
    }
    normal[0] = f.poly.normal.x;
    normal[1] = f.poly.normal.y;
    normal[2] = f.poly.normal.z;
    return n;
}

int32_t vref_edge_export(void* h, int32_t idx, char* id, int32_t idcap, double* ab) {
    const R::Edge& e = static_cast<RefScene*>(h)->scene.edges().at(static_cast<size_t>(idx));
    std::snprintf(id, static_cast<size_t>(idcap), "%s", e.id.c_str());
    ab[0] = e.a.x; ab[1] = e.a.y; ab[2] = e.a.z;
    ab[3] = e.b.x; ab[4] = e.b.y; ab[5] = e.b.z;
    return 0;
}

// ---------------------------------------------------------------------------
// (1) occlusion_judgment (proj/src/vismatrix.cpp:253-302), prefilter pieces
// ---------------------------------------------------------------------------

// Returns kind 0 Visible / 1 PartiallyVisible / 2 Occluded, or -1 on error.
// Blockers are returned as face indices in the reference's (string-sorted) order.
int32_t vref_occlusion(void* h, int32_t i, int32_t j, int32_t* blockers, int32_t cap,
                       int32_t* nblk) {
    try {
        const R::Scene& s = static_cast<RefScene*>(h)->scene;
        const R::OcclusionVerdict v = R::occlusion_judgment(s.face(i), s.face(j), s);
        *nblk = static_cast<int32_t>(v.blockers.size());
        for (int32_t k = 0; k < *nblk && k < cap; ++k) blockers[k] = s.face(v.blockers[k]).index;
        return static_cast<int32_t>(v.kind);
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// Batch verdict kinds over a pair list on `threads` workers (atomic counter,
// the reference's own scheduling pattern, proj/src/vismatrix.cpp:654-667).
int32_t vref_occlusion_batch(void* h, int64_t npairs, const int32_t* pi, const int32_t* pj,
                             int8_t* kind, int32_t threads) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    std::atomic<int64_t> next{0};
    std::atomic<int> bad{0};
    auto work = [&]() {
        for (int64_t k = next.fetch_add(1); k < npairs; k = next.fetch_add(1)) {
            try {
                kind[k] = static_cast<int8_t>(
                    R::occlusion_judgment(s.face(pi[k]), s.face(pj[k]), s).kind);
            } catch (...) {
                kind[k] = -1;
                bad = 1;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return bad.load();
}

int32_t vref_mutually_front(void* h, int32_t i, int32_t j) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    return R::mutually_front(s.face(i), s.face(j)) ? 1 : 0;
}

// Bitmask of required planes (bit 0 XY, 1 YZ, 2 XZ), proj/src/vismatrix.cpp:171-181.
int32_t vref_required_planes(void* h, int32_t i, int32_t j) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    int32_t m = 0;
    for (R::PlaneTag t : R::required_planes(s.face(i), s.face(j))) m |= 1 << static_cast<int>(t);
    return m;
}

// build_matrix's triple_ext feasibility (proj/src/vismatrix.cpp:715-751) for one
// triple p -> t -> a of admitted pairs, through the reference's public
// chain_triple_feasible / required_planes / second_order_check. The matrix
// second_order_check consults only needs the two order-1 legs, so a minimal
// one with those entries stands in for the full build.
// chain_triple_feasible alone (proj/src/vismatrix.cpp:457-476)
int32_t vref_chain_triple_feasible(void* h, int32_t p, int32_t t, int32_t a) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    return R::chain_triple_feasible(s.face(p), s.face(t), s.face(a)) ? 1 : 0;
}

// the K7 filter: chain_triple_feasible and second_order_check != None per shared plane
int32_t vref_triple_feasible(void* h, int32_t p, int32_t t, int32_t a) {
    try {
        const R::Scene& s = static_cast<RefScene*>(h)->scene;
        const R::Face& fp = s.face(p);
        const R::Face& ft = s.face(t);
        const R::Face& fa = s.face(a);
        if (!R::chain_triple_feasible(fp, ft, fa)) return 0;
        R::InterVisMatrix m;
        auto add_leg = [&](const R::Face& x, const R::Face& y) {
            for (R::PlaneTag pl : R::required_planes(x, y)) {
                R::InterVisEntry e;
                e.order = 1;
                e.ref = x.id;
                e.aim = y.id;
                e.relation.plane = pl;
                e.relation.chain = {x.id, y.id};
                m.add(e);
            }
        };
        add_leg(fp, ft);
        add_leg(ft, fa);
        for (R::PlaneTag pl : R::required_planes(ft, fa)) {
            if (!m.find(1, fp.id, ft.id, pl)) continue;
            if (R::second_order_check(fp, ft, fa, m, pl).verdict == R::ChainVerdict::None) return 0;
        }
        return 1;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// plane_segment (proj/src/scene.cpp:213-254): returns 1 and a,b,normal (6 doubles) if present.
int32_t vref_plane_segment(void* h, int32_t i, int32_t plane, double* out6) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    const auto seg = R::plane_segment(s.face(i), static_cast<R::PlaneTag>(plane));
    if (!seg) return 0;
    out6[0] = seg->a.x; out6[1] = seg->a.y; out6[2] = seg->b.x; out6[3] = seg->b.y;
    out6[4] = seg->normal.x; out6[5] = seg->normal.y;
    return 1;
}

// segment_face_intersection (proj/src/geom.cpp:169-180) on a scene face.
int32_t vref_segment_hits_face(void* h, const double* a, const double* b, int32_t face) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    return R::segment_face_intersection({a[0], a[1], a[2]}, {b[0], b[1], b[2]}, s.face(face).poly)
               ? 1
               : 0;
}

// sightline_clear semantics (proj/src/vistable.cpp:38-44, skip = none) for a
// batch of segments: blocked[k] = some face's segment_face_intersection hits
// (a_k, b_k). Host thread pool.
int32_t vref_segments_blocked(void* h, int64_t n, const double* a, const double* b, uint8_t* blocked,
                              int32_t threads) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    std::atomic<int64_t> next{0};
    auto work = [&]() {
        for (int64_t k = next.fetch_add(1); k < n; k = next.fetch_add(1)) {
            const R::Vec3 pa{a[3 * k], a[3 * k + 1], a[3 * k + 2]}, pb{b[3 * k], b[3 * k + 1], b[3 * k + 2]};
            uint8_t hit = 0;
            for (const R::Face* f : s.faces())
                if (R::segment_face_intersection(pa, pb, f->poly)) {
                    hit = 1;
                    break;
                }
            blocked[k] = hit;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return 0;
}

// ---------------------------------------------------------------------------
// build_matrix (proj/src/vismatrix.cpp:638-799) — entries exported flat
// ---------------------------------------------------------------------------


void* vref_build_matrix(void* h, int32_t order) {
    try {
        const R::Scene& s = static_cast<RefScene*>(h)->scene;
        return new R::InterVisMatrix(R::build_matrix(s, order));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void vref_matrix_free(void* m) { delete static_cast<R::InterVisMatrix*>(m); }
void vref_matrix_set_max_order(void* m, int32_t order) {
    static_cast<R::InterVisMatrix*>(m)->set_max_order(order);
}

int64_t vref_matrix_size(void* m) {
    return static_cast<int64_t>(static_cast<R::InterVisMatrix*>(m)->entries().size());
}

// the chains (face indices) of every entry of one order, flat [k][order + 1];
// out == NULL: count only. Bulk form of vref_matrix_entry for big matrices.
int64_t vref_matrix_chains(void* h, void* m, int32_t order, int32_t* out, int64_t cap) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    int64_t c = 0;
    for (const R::InterVisEntry& e : static_cast<R::InterVisMatrix*>(m)->entries()) {
        if (e.order != order) continue;
        if (out && c < cap)
            for (size_t q = 0; q < e.relation.chain.size() && q <= static_cast<size_t>(order); ++q)
                out[c * (order + 1) + static_cast<int64_t>(q)] = s.face(e.relation.chain[q]).index;
        ++c;
    }
    return c;
}

int32_t vref_matrix_entry(void* h, void* m, int64_t k, vref_entry* out) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    const R::InterVisEntry& e = static_cast<R::InterVisMatrix*>(m)->entries().at(static_cast<size_t>(k));
    std::memset(out, 0, sizeof(*out));
    out->order = e.order;
    out->chain_len = static_cast<int32_t>(e.relation.chain.size());
    for (int32_t c = 0; c < out->chain_len && c < 5; ++c) out->chain[c] = s.face(e.relation.chain[c]).index;
    out->plane = static_cast<int32_t>(e.relation.plane);
    out->kind = e.relation.kind == R::RelationKind::Parallel ? 0 : 1;
    out->verdict = e.verdict == R::ChainVerdict::Full ? 0 : 1;
    auto rec = [](const R::AngleRecord& r, double* d) {
        d[0] = r.vertex.x; d[1] = r.vertex.y; d[2] = r.low; d[3] = r.high;
        d[4] = r.ref_dir.x; d[5] = r.ref_dir.y;
    };
    rec(e.ranges.at_a, out->ranges);
    rec(e.ranges.at_b, out->ranges + 6);
    std::snprintf(out->edge_a, sizeof(out->edge_a), "%s", e.ranges.at_a.edge_id.c_str());
    std::snprintf(out->edge_b, sizeof(out->edge_b), "%s", e.ranges.at_b.edge_id.c_str());
    if (e.criterion) {
        out->has_criterion = 1;
        out->criterion[0] = e.criterion->at_a.low;
        out->criterion[1] = e.criterion->at_a.high;
        out->criterion[2] = e.criterion->at_b.low;
        out->criterion[3] = e.criterion->at_b.high;
    }
    out->nsub = static_cast<int32_t>(e.subranges.size());
    for (int32_t q = 0; q < out->nsub && q < 4; ++q) {
        out->sub[2 * q] = e.subranges[q][0];
        out->sub[2 * q + 1] = e.subranges[q][1];
    }
    out->nblockers = static_cast<int32_t>(e.blockers.size());
    for (int32_t q = 0; q < out->nblockers && q < 64; ++q) out->blockers[q] = s.face(e.blockers[q]).index;
    out->naim_image = static_cast<int32_t>(e.aim_image.size());
    for (int32_t q = 0; q < out->naim_image && q < 8; ++q) {
        out->aim_image[3 * q] = e.aim_image[q].x;
        out->aim_image[3 * q + 1] = e.aim_image[q].y;
        out->aim_image[3 * q + 2] = e.aim_image[q].z;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// (2) illuminated_region (proj/src/vistable.cpp:287-334)
// ---------------------------------------------------------------------------


int32_t vref_illuminated_region(void* h, const double* src, int32_t face, vref_region* out) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    std::memset(out, 0, sizeof(*out));
    try {
        const auto reg = R::illuminated_region({src[0], src[1], src[2]}, s.face(face), s);
        if (!reg) return 0;
        out->present = 1;
        out->nplanes = static_cast<int32_t>(reg->planes.size());
        for (int32_t p = 0; p < out->nplanes; ++p) {
            const R::PlaneIllumination& pi = reg->planes[static_cast<size_t>(p)];
            out->plane[p] = static_cast<int32_t>(pi.plane);
            out->clipped[p] = pi.clipped ? 1 : 0;
            out->sub[2 * p] = pi.sub[0];
            out->sub[2 * p + 1] = pi.sub[1];
            out->image[2 * p] = pi.image.x;
            out->image[2 * p + 1] = pi.image.y;
            out->sub_ab[4 * p] = pi.sub_a.x;
            out->sub_ab[4 * p + 1] = pi.sub_a.y;
            out->sub_ab[4 * p + 2] = pi.sub_b.x;
            out->sub_ab[4 * p + 3] = pi.sub_b.y;
            out->angles[4 * p] = pi.alpha_full;
            out->angles[4 * p + 1] = pi.beta_full;
            out->angles[4 * p + 2] = pi.alpha;
            out->angles[4 * p + 3] = pi.beta;
        }
        return 0;
    } catch (const R::VisibilityError& e) {
        out->present = -1;
        g_err = e.what();
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 5);
    }
}

// Batch over (source, face) pairs on a thread pool; VisibilityError -> present = -1.
int32_t vref_regions_batch(void* h, int64_t n, const double* src, const int32_t* face,
                           vref_region* out, int32_t threads) {
    std::atomic<int64_t> next{0};
    auto work = [&]() {
        for (int64_t k = next.fetch_add(1); k < n; k = next.fetch_add(1)) {
            vref_illuminated_region(h, src + 3 * k, face[k], out + k);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return 0;
}

// point_vis_table (proj/src/vistable.cpp:478-521): rows flattened.

int64_t vref_point_vis_table(void* h, void* m, const double* src, int32_t max_order, vref_row* rows,
                             int64_t cap) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    try {
        const auto t = R::point_vis_table({src[0], src[1], src[2]},
                                          *static_cast<R::InterVisMatrix*>(m), s, max_order);
        const int64_t n = static_cast<int64_t>(t.size());
        for (int64_t k = 0; k < n && k < cap; ++k) {
            const R::VisTableEntry& e = t[static_cast<size_t>(k)];
            vref_row& r = rows[k];
            std::memset(&r, 0, sizeof(r));
            r.order = e.order;
            r.chain_len = static_cast<int32_t>(e.chain.size());
            for (int32_t c = 0; c < r.chain_len && c < 4; ++c) r.chain[c] = s.face(e.chain[c]).index;
            r.aim = s.face(e.aim).index;
            r.plane = static_cast<int32_t>(e.plane);
            r.verdict = e.verdict == R::ChainVerdict::Full ? 0 : 1;
            std::snprintf(r.ref_display, sizeof(r.ref_display), "%s", e.ref_display.c_str());
            std::snprintf(r.aim_display, sizeof(r.aim_display), "%s", e.aim_display.c_str());
            std::snprintf(r.parent_display, sizeof(r.parent_display), "%s", e.parent_display.c_str());
        }
        return n;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// ---------------------------------------------------------------------------
// (3) TraceAccelerator / brute_force_trace / image_tree (proj/src/raytracer.cpp)
// ---------------------------------------------------------------------------

void* vref_accel_create(void* h, void* m, int32_t max_refl) {
    try {
        return new R::TraceAccelerator(static_cast<RefScene*>(h)->scene,
                                       *static_cast<R::InterVisMatrix*>(m), max_refl);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void vref_accel_free(void* a) { delete static_cast<R::TraceAccelerator*>(a); }


static int64_t export_paths(const R::Scene& s, const std::vector<R::Path>& paths, vref_path* out,
                            int64_t cap) {
    const int64_t n = static_cast<int64_t>(paths.size());
    for (int64_t k = 0; k < n && k < cap; ++k) {
        const R::Path& p = paths[static_cast<size_t>(k)];
        vref_path& o = out[k];
        std::memset(&o, 0, sizeof(o));
        o.ninter = static_cast<int32_t>(p.interactions.size());
        for (int32_t q = 0; q < o.ninter && q < 6; ++q) {
            const auto& it = p.interactions[static_cast<size_t>(q)];
            o.is_diff[q] = it.kind == R::InteractionKind::Diffraction ? 1 : 0;
            o.face[q] = o.is_diff[q] ? -1 : s.face(it.id).index;
        }
        for (size_t q = 0; q < p.points.size() && q < 8; ++q) {
            o.points[3 * q] = p.points[q].x;
            o.points[3 * q + 1] = p.points[q].y;
            o.points[3 * q + 2] = p.points[q].z;
        }
        o.length = p.length;
        o.delay = p.delay;
        std::snprintf(o.identity, sizeof(o.identity), "%s", p.identity().c_str());
    }
    return n;
}

// stats: nodes_expanded, sequences_checked, occlusion_tests, paths_found
int64_t vref_accel_trace(void* h, void* a, const double* tx, const double* rx, int32_t diffraction,
                         vref_path* out, int64_t cap, int64_t* stats) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    try {
        R::TraceStats st;
        const auto paths = static_cast<R::TraceAccelerator*>(a)->trace(
            {tx[0], tx[1], tx[2]}, {rx[0], rx[1], rx[2]}, diffraction != 0, &st);
        if (stats) {
            stats[0] = st.nodes_expanded;
            stats[1] = st.sequences_checked;
            stats[2] = st.occlusion_tests;
            stats[3] = st.paths_found;
        }
        return export_paths(s, paths, out, cap);
    } catch (const std::exception& e) {
        return fail(e, -1 - error_code(e));
    }
}

int64_t vref_brute_trace(void* h, const double* tx, const double* rx, int32_t max_refl,
                         int32_t diffraction, vref_path* out, int64_t cap, int64_t* stats) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    try {
        R::TraceStats st;
        const auto paths = R::brute_force_trace(s, {tx[0], tx[1], tx[2]}, {rx[0], rx[1], rx[2]},
                                                max_refl, diffraction != 0, &st);
        if (stats) {
            stats[0] = st.nodes_expanded;
            stats[1] = st.sequences_checked;
            stats[2] = st.occlusion_tests;
            stats[3] = st.paths_found;
        }
        return export_paths(s, paths, out, cap);
    } catch (const std::exception& e) {
        return fail(e, -1 - error_code(e));
    }
}

// Batch of accelerated traces over snapshots on a thread pool (trace() is
// const and re-entrant, proj/include/rt/raytracer.hpp:92-94). Returns total
// path count; per-snapshot counts in npaths[k]; node counts in nodes[k].
int64_t vref_accel_trace_batch(void* h, void* a, int64_t n, const double* tx, const double* rx,
                               int32_t rx_fixed, int32_t threads, int64_t* npaths, int64_t* nodes) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    (void)s;
    std::atomic<int64_t> next{0};
    std::atomic<int64_t> total{0};
    auto work = [&]() {
        for (int64_t k = next.fetch_add(1); k < n; k = next.fetch_add(1)) {
            const double* r = rx_fixed ? rx : rx + 3 * k;
            try {
                R::TraceStats st;
                const auto paths = static_cast<R::TraceAccelerator*>(a)->trace(
                    {tx[3 * k], tx[3 * k + 1], tx[3 * k + 2]}, {r[0], r[1], r[2]}, false, &st);
                npaths[k] = static_cast<int64_t>(paths.size());
                nodes[k] = st.nodes_expanded;
                total += npaths[k];
            } catch (...) {
                npaths[k] = -1;
                nodes[k] = -1;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return total.load();
}

// image_tree (proj/src/raytracer.cpp:458-486): node face index, parent, depth, image.
int64_t vref_image_tree(void* h, const double* src, int32_t depth, int32_t* face, int32_t* parent,
                        int32_t* dep, double* image, int64_t cap) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    const auto t = R::image_tree(s, {src[0], src[1], src[2]}, depth);
    const int64_t n = static_cast<int64_t>(t.size());
    for (int64_t k = 0; k < n && k < cap; ++k) {
        face[k] = s.face(t[static_cast<size_t>(k)].face).index;
        parent[k] = t[static_cast<size_t>(k)].parent;
        dep[k] = t[static_cast<size_t>(k)].depth;
        image[3 * k] = t[static_cast<size_t>(k)].image.x;
        image[3 * k + 1] = t[static_cast<size_t>(k)].image.y;
        image[3 * k + 2] = t[static_cast<size_t>(k)].image.z;
    }
    return n;
}

// dynamic_trace against a fixed receiver (proj/src/raytracer.cpp:590-643):
// per sample s, segment, retraced flag and the paths (identity, points, length)
// flattened; waypoints [nwp][3] with speed 1 m/s.
typedef struct {
    double s;
    int32_t segment;
    int32_t retraced;
    int32_t npaths;
    int32_t first;   // index of its first path in the path array
} vref_dyn_sample;

int64_t vref_dynamic_trace(void* h, void* m, int32_t nwp, const double* wp, const double* rx, int32_t max_refl,
                           int32_t diffraction, double step, vref_dyn_sample* samples, int64_t scap,
                           vref_path* paths, int64_t pcap, int64_t* npaths_out) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    try {
        R::Trajectory traj;
        for (int32_t k = 0; k < nwp; ++k) traj.waypoints.push_back({wp[3 * k], wp[3 * k + 1], wp[3 * k + 2]});
        traj.speeds.assign(static_cast<size_t>(nwp > 1 ? nwp - 1 : 1), 1.0);
        const auto res = R::dynamic_trace(s, *static_cast<R::InterVisMatrix*>(m), traj, {rx[0], rx[1], rx[2]},
                                          max_refl, diffraction != 0, step);
        int64_t np = 0;
        const int64_t ns = static_cast<int64_t>(res.samples.size());
        for (int64_t k = 0; k < ns; ++k) {
            const auto& smp = res.samples[static_cast<size_t>(k)];
            if (k < scap) {
                samples[k].s = smp.s;
                samples[k].segment = smp.segment;
                samples[k].retraced = smp.retraced ? 1 : 0;
                samples[k].npaths = static_cast<int32_t>(smp.paths.size());
                samples[k].first = static_cast<int32_t>(np);
            }
            for (const auto& p : smp.paths) {
                if (np < pcap) {
                    vref_path& o = paths[np];
                    std::memset(&o, 0, sizeof(o));
                    o.ninter = static_cast<int32_t>(p.interactions.size());
                    for (size_t q = 0; q < p.points.size() && q < 8; ++q) {
                        o.points[3 * q] = p.points[q].x;
                        o.points[3 * q + 1] = p.points[q].y;
                        o.points[3 * q + 2] = p.points[q].z;
                    }
                    o.length = p.length;
                    o.delay = p.delay;
                    std::snprintf(o.identity, sizeof(o.identity), "%s", p.identity().c_str());
                }
                ++np;
            }
        }
        *npaths_out = np;
        return ns;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// Face material parameters (permittivity, conductivity) and edge faces, for
// the EM consumer (proj/src/em.cpp).
int32_t vref_face_material(void* h, int32_t idx, double* eps_sigma) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    try {
        const R::Material& m = s.material(s.face(idx).material);
        eps_sigma[0] = m.permittivity;
        eps_sigma[1] = m.conductivity;
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

int32_t vref_edge_faces(void* h, int32_t idx, int32_t* faces) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    const R::Edge& e = s.edges().at(static_cast<size_t>(idx));
    faces[0] = s.face(e.faces[0]).index;
    faces[1] = s.face(e.faces[1]).index;
    return 0;
}

// ray_gains + channel_stats (proj/src/em.cpp:194-277) of an accelerated trace:
// per path amplitude (re, im) and delay (path order = the trace's), plus
// [outage, path_loss_db, rms_delay_spread].
int64_t vref_trace_em(void* h, void* a, const double* tx, const double* rx, int32_t diffraction, double freq,
                      double tx_gain, double rx_gain, int32_t tm, double* amp, double* delay, double* stats3,
                      int64_t cap) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    try {
        const auto paths = static_cast<R::TraceAccelerator*>(a)->trace({tx[0], tx[1], tx[2]}, {rx[0], rx[1], rx[2]},
                                                                       diffraction != 0, nullptr);
        R::EmConfig cfg;
        cfg.frequency = freq;
        cfg.tx_gain_dbi = tx_gain;
        cfg.rx_gain_dbi = rx_gain;
        cfg.polarization = tm ? R::Polarization::TM : R::Polarization::TE;
        const auto rays = R::ray_gains(s, paths, cfg);
        const auto st = R::channel_stats(rays);
        const int64_t n = static_cast<int64_t>(rays.size());
        for (int64_t k = 0; k < n && k < cap; ++k) {
            amp[2 * k] = rays[static_cast<size_t>(k)].amplitude.real();
            amp[2 * k + 1] = rays[static_cast<size_t>(k)].amplitude.imag();
            delay[k] = rays[static_cast<size_t>(k)].delay;
        }
        stats3[0] = st.outage ? 1.0 : 0.0;
        stats3[1] = st.path_loss_db;
        stats3[2] = st.rms_delay_spread;
        return n;
    } catch (const std::exception& e) {
        return fail(e, -1 - error_code(e));
    }
}

// closest_diffraction_edge (proj/src/vistable.cpp:545-561): edge index or -1.
int32_t vref_closest_edge(void* h, const double* rx) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    const auto e = R::closest_diffraction_edge({rx[0], rx[1], rx[2]}, s);
    if (!e) return -1;
    const auto& edges = s.edges();
    for (size_t k = 0; k < edges.size(); ++k)
        if (edges[k].id == e->id) return static_cast<int32_t>(k);
    return -2;
}

// trajectory_vis_table (proj/src/vistable.cpp:822-960): rows flattened.
// waypoints: [nwp][3]; speeds are irrelevant to the table (1 m/s).

int64_t vref_trajectory_table(void* h, void* m, int32_t nwp, const double* wp, int32_t max_order,
                              vref_mobile_row* rows, int64_t cap) {
    const R::Scene& s = static_cast<RefScene*>(h)->scene;
    try {
        R::Trajectory traj;
        for (int32_t k = 0; k < nwp; ++k) traj.waypoints.push_back({wp[3 * k], wp[3 * k + 1], wp[3 * k + 2]});
        traj.speeds.assign(static_cast<size_t>(nwp > 1 ? nwp - 1 : 1), 1.0);
        const auto t = R::trajectory_vis_table(traj, *static_cast<R::InterVisMatrix*>(m), s, max_order);
        const int64_t n = static_cast<int64_t>(t.size());
        for (int64_t k = 0; k < n && k < cap; ++k) {
            const R::MobileVisEntry& e = t[static_cast<size_t>(k)];
            vref_mobile_row& r = rows[k];
            std::memset(&r, 0, sizeof(r));
            r.order = e.order;
            r.s_start = e.s_start;
            r.s_end = e.s_end;
            std::snprintf(r.node, sizeof(r.node), "%s", e.node.c_str());
            std::snprintf(r.node_display, sizeof(r.node_display), "%s", e.node_display.c_str());
            std::snprintf(r.label_start, sizeof(r.label_start), "%s", e.label_start.c_str());
            std::snprintf(r.label_end, sizeof(r.label_end), "%s", e.label_end.c_str());
            std::snprintf(r.parent, sizeof(r.parent), "%s", e.parent.c_str());
            std::snprintf(r.blockage, sizeof(r.blockage), "%s", e.blockage.c_str());
        }
        return n;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

}  // extern "C"
