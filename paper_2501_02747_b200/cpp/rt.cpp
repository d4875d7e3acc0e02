// visrt-b200 C++ drop-in layer (see rt.hpp). Every geometric decision comes
// from the C-ABI (GPU); this file only materialises the reference's records:
// ids, angle records (atan2 on the host, as the reference), aim images,
// ordering. Compiled with -ffp-contract=off.
#include "rt.hpp"

#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <cstring>
#include <set>
#include <unordered_set>

#include "../../include/visrt.h"

#include <fstream>

#include <json.hpp>   // nlohmann 3.11 (the image's vendored copy; host I/O only)

namespace rt {
namespace {

[[noreturn]] void fail(int rc) {
    const std::string msg = visrt_last_error();
    if (rc == VISRT_E_VISIBILITY) throw VisibilityError(msg);
    if (rc == VISRT_E_PLACEMENT) throw PlacementError(msg);
    if (rc == VISRT_E_SCENE) throw SceneError(msg);
    throw std::runtime_error("visrt: " + msg);
}
void check(int rc) {
    if (rc != VISRT_OK) fail(rc);
}

double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// string order -> integer ranks (the C-ABI takes the reference's sort keys as ranks)
template <class T>
std::map<T, int32_t> ranks_of(std::vector<T> v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    std::map<T, int32_t> r;
    for (size_t k = 0; k < v.size(); ++k) r.emplace(v[k], static_cast<int32_t>(k));
    return r;
}
std::string building_of(const Face& f) { return f.building.empty() ? "ground" : f.building; }
double norm(const Vec3& a) { return std::sqrt(dot(a, a)); }
double dot2(const Vec2& a, const Vec2& b) { return a.x * b.x + a.y * b.y; }
double cross2(const Vec2& a, const Vec2& b) { return a.x * b.y - a.y * b.x; }
double norm2(const Vec2& a) { return std::sqrt(dot2(a, a)); }
Vec2 sub2(const Vec2& a, const Vec2& b) { return {a.x - b.x, a.y - b.y}; }
Vec2 project(const Vec3& p, PlaneTag t) {
    if (t == PlaneTag::XY) return {p.x, p.y};
    if (t == PlaneTag::YZ) return {p.y, p.z};
    return {p.x, p.z};
}
double signed_distance(const Face& f, const Vec3& p) { return dot(p - f.poly.pts.front(), f.poly.normal); }
Vec3 mirror(const Face& f, const Vec3& p) { return p - f.poly.normal * (2.0 * signed_distance(f, p)); }
Orientation classify(const Vec3& n) {   // src/scene.cpp:19-24
    const double ax = std::abs(n.x), ay = std::abs(n.y), az = std::abs(n.z);
    if (ax <= 1e-9 && ay <= 1e-9) return Orientation::Horizontal;
    if (az <= 1e-9) return Orientation::Vertical;
    return Orientation::Oblique;
}

// oriented_angle_deg / clamp_visibility_angle, src/geom.cpp:64-77
double oriented_angle(const Vec2& d, const Vec2& n, const Vec2& v) {
    constexpr double kRad2Deg = 180.0 / 3.14159265358979323846;
    const double s = cross2(d, n) >= 0.0 ? 1.0 : -1.0;
    double a = std::atan2(s * cross2(d, v), dot2(d, v)) * kRad2Deg;
    if (a < 0.0) a += 360.0;
    if (a >= 360.0) a -= 360.0;
    return a;
}
double clamp_angle(double a) { return a < 180.0 ? a : 0.0; }

struct Segs {   // plane segments of every face, from the C-ABI ingest
    std::vector<double> seg;
    std::vector<int32_t> ok;
    bool has(int f, int pl) const { return ok[3 * static_cast<size_t>(f) + pl] != 0; }
    PlaneSegment get(int f, int pl) const {
        const double* s = &seg[(static_cast<size_t>(f) * 3 + pl) * 6];
        return {{s[0], s[1]}, {s[2], s[3]}, {s[4], s[5]}};
    }
};

Segs scene_segs(const Scene& sc) {
    Segs s;
    const int n = static_cast<int>(sc.faces().size());
    s.seg.resize(static_cast<size_t>(n) * 18);
    s.ok.resize(static_cast<size_t>(n) * 3);
    check(visrt_scene_ingest(sc.device_scene(), nullptr, nullptr, s.seg.data(), s.ok.data()));
    return s;
}

// required_planes, src/vismatrix.cpp:171-181
std::vector<PlaneTag> required_planes(const Segs& s, int i, int j) {
    std::vector<PlaneTag> out;
    for (int pl = 0; pl < 3; ++pl) {
        if (!s.has(i, pl) || !s.has(j, pl)) continue;
        const double d = std::abs(dot2(s.get(i, pl).normal, s.get(j, pl).normal));
        if (d >= 1.0 - 1e-9 || d <= 1e-9) out.push_back(static_cast<PlaneTag>(pl));
    }
    return out;
}

// bounding_edge_id, src/vismatrix.cpp:316-330
std::string bounding_edge_id(const Scene& sc, const Face& face, PlaneTag plane, const Vec2& endpoint) {
    if (face.building.empty()) return "";
    for (const Edge& e : sc.edges()) {
        if (e.building != face.building) continue;
        if (std::find(e.faces.begin(), e.faces.end(), face.id) == e.faces.end()) continue;
        const Vec2 pa = project(e.a, plane), pb = project(e.b, plane);
        if (norm2(sub2(pa, endpoint)) <= 1e-9 && norm2(sub2(pb, endpoint)) <= 1e-9) return e.id;
    }
    return "";
}

// angle_record / first_order_ranges / clamp_complement, src/vismatrix.cpp:332-385
AngleRecord angle_record(const Scene& sc, const Face& ref, PlaneTag plane, const Vec2& at, const Vec2& other,
                         const Vec2& outward, const PlaneSegment& aim) {
    AngleRecord rec;
    rec.vertex = at;
    rec.outward = outward;
    const Vec2 d = sub2(other, at);
    const double inv = 1.0 / norm2(d);
    rec.ref_dir = {d.x * inv, d.y * inv};
    rec.edge_id = bounding_edge_id(sc, ref, plane, at);
    auto angle_to = [&](const Vec2& t) {
        const Vec2 v = sub2(t, at);
        if (norm2(v) <= kEps) return 0.0;
        return clamp_angle(oriented_angle(rec.ref_dir, outward, v));
    };
    const double a1 = angle_to(aim.a), a2 = angle_to(aim.b);
    rec.low = std::min(a1, a2);
    rec.high = std::max(a1, a2);
    return rec;
}
AngularBouncingRange first_order_ranges(const Scene& sc, const Segs& s, int ref, int aim, PlaneTag plane) {
    const PlaneSegment sr = s.get(ref, static_cast<int>(plane)), sa = s.get(aim, static_cast<int>(plane));
    const Face& f = sc.face(ref);
    return {angle_record(sc, f, plane, sr.a, sr.b, sr.normal, sa), angle_record(sc, f, plane, sr.b, sr.a, sr.normal, sa)};
}
AngularBouncingRange clamp_complement(const AngularBouncingRange& r) {
    auto flip = [](const AngleRecord& rec) {
        AngleRecord out = rec;
        const double a = clamp_angle(180.0 - rec.low), b = clamp_angle(180.0 - rec.high);
        out.low = std::min(a, b);
        out.high = std::max(a, b);
        return out;
    };
    return {flip(r.at_a), flip(r.at_b)};
}
InterfaceRelation relation(const Scene& sc, const Segs& s, int ref, int aim, PlaneTag plane) {
    const double d = std::abs(dot2(s.get(ref, static_cast<int>(plane)).normal, s.get(aim, static_cast<int>(plane)).normal));
    InterfaceRelation r;
    r.plane = plane;
    r.chain = {sc.face(ref).id, sc.face(aim).id};
    r.chain_orientations = {sc.face(ref).orientation, sc.face(aim).orientation};
    r.kind = d >= 1.0 - 1e-9 ? RelationKind::Parallel : RelationKind::Perpendicular;
    return r;
}
std::vector<Vec3> chain_image(const Scene& sc, const std::vector<int>& chain) {   // 306-314
    const Face& aim = sc.face(chain.back());
    std::vector<Vec3> img(aim.poly.pts.begin(), aim.poly.pts.end());
    for (size_t k = chain.size() - 1; k-- > 0;)
        for (Vec3& p : img) p = mirror(sc.face(chain[k]), p);
    return img;
}

// second_order_check verdict + reachable set (src/vismatrix.cpp:43-147, 387-455):
// the host re-derives the record fields of a chain the GPU found feasible.
using Interval = std::array<double, 2>;
using ISet = std::vector<Interval>;
ISet normalize(ISet s) {
    std::sort(s.begin(), s.end());
    ISet out;
    for (const Interval& iv : s) {
        if (iv[1] - iv[0] < 0) continue;
        if (!out.empty() && iv[0] <= out.back()[1] + 1e-15) out.back()[1] = std::max(out.back()[1], iv[1]);
        else out.push_back(iv);
    }
    return out;
}
ISet halfline(double a, double b, bool leq, double lo, double hi) {
    if (!leq) {
        a = -a;
        b = -b;
    }
    if (std::abs(a) < 1e-300) return b <= 0 ? ISet{{lo, hi}} : ISet{};
    const double t = -b / a;
    if (a > 0) return t < lo ? ISet{} : ISet{{lo, std::min(t, hi)}};
    return t > hi ? ISet{} : ISet{{std::max(t, lo), hi}};
}
bool clip_upper(const Vec2& p0, const Vec2& p1, double& lo, double& hi) {
    lo = 0.0;
    hi = 1.0;
    const double dy = p1.y - p0.y;
    if (std::abs(dy) < 1e-300) return p0.y >= -kEps;
    const double tc = -p0.y / dy;
    if (dy > 0) lo = std::max(0.0, tc);
    else hi = std::min(1.0, tc);
    return hi - lo > 1e-12;
}
ChainVerdict second_order(const Segs& s, int o, int m, int t, PlaneTag plane, ISet& reach_out) {
    const int pl = static_cast<int>(plane);
    const PlaneSegment so = s.get(o, pl), sm = s.get(m, pl), st = s.get(t, pl);
    Vec2 origin = sm.a;
    const Vec2 d = sub2(sm.b, sm.a);
    const double inv = 1.0 / norm2(d);
    Vec2 ux{d.x * inv, d.y * inv};
    if (cross2(ux, sm.normal) < 0) {
        origin = sm.b;
        ux = {ux.x * -1.0, ux.y * -1.0};
    }
    auto map = [&](const Vec2& p) { const Vec2 r = sub2(p, origin); return Vec2{dot2(r, ux), dot2(r, sm.normal)}; };
    const double length = norm2(sub2(sm.b, sm.a));
    Vec2 p0 = map(so.a), p1 = map(so.b);
    double lo, hi;
    if (!clip_upper(p0, p1, lo, hi)) return ChainVerdict::None;
    const Vec2 q0{p0.x + lo * (p1.x - p0.x), p0.y + lo * (p1.y - p0.y)};
    const Vec2 q1{p0.x + hi * (p1.x - p0.x), p0.y + hi * (p1.y - p0.y)};
    p0 = q0;
    p1 = q1;
    const Vec2 c0 = map(st.a), c1 = map(st.b);
    double dlo, dhi;
    if (!clip_upper(c0, c1, dlo, dhi)) return ChainVerdict::None;
    const Vec2 m0{c0.x, -c0.y}, md{c1.x - c0.x, -(c1.y - c0.y)};
    auto cond = [&](const Vec2& p, double bound, bool leq) {
        const double a_num = md.x * p.y - p.x * md.y, b_num = m0.x * p.y - p.x * m0.y;
        const double a_den = -md.y, b_den = p.y - m0.y;
        return halfline(a_num - bound * a_den, b_num - bound * b_den, leq, dlo, dhi);
    };
    ISet right = cond(p0, length, true), r1 = cond(p1, length, true);
    right.insert(right.end(), r1.begin(), r1.end());
    right = normalize(right);
    ISet left = cond(p0, 0.0, false), l1 = cond(p1, 0.0, false);
    left.insert(left.end(), l1.begin(), l1.end());
    left = normalize(left);
    ISet reach;
    for (const Interval& x : right)
        for (const Interval& y : left) {
            const double a = std::max(x[0], y[0]), b = std::min(x[1], y[1]);
            if (a <= b) reach.push_back({a, b});
        }
    reach = normalize(reach);
    double len = 0;
    for (const Interval& iv : reach) len += iv[1] - iv[0];
    if (len <= 1e-12) return ChainVerdict::None;
    reach_out = reach;
    if (reach.size() == 1 && reach.front()[0] <= 1e-9 && reach.front()[1] >= 1.0 - 1e-9) {
        reach_out.clear();
        return ChainVerdict::Full;
    }
    return ChainVerdict::Partial;
}

}  // namespace

// ---------------------------------------------------------------------------
ConvexPolygon ConvexPolygon::from_points(std::vector<Vec3> pts) {
    if (pts.size() < 3) throw std::invalid_argument("polygon needs at least three vertices");
    Vec3 n{0, 0, 0};
    for (size_t i = 0; i < pts.size(); ++i) {   // Newell, src/geom.cpp:126-140
        const Vec3& a = pts[i];
        const Vec3& b = pts[(i + 1) % pts.size()];
        n.x += (a.y - b.y) * (a.z + b.z);
        n.y += (a.z - b.z) * (a.x + b.x);
        n.z += (a.x - b.x) * (a.y + b.y);
    }
    const double len = norm(n);
    if (len < kEps) throw std::invalid_argument("cannot normalize zero-length vector");
    ConvexPolygon p;
    p.normal = {n.x / len, n.y / len, n.z / len};
    p.pts = std::move(pts);
    return p;
}

namespace {
// Face -> owning Scene, for the reference's scene-less predicates that need
// the device scene (chain_triple_feasible)
std::mutex g_owner_mu;
std::unordered_map<const Face*, const Scene*> g_owner;
void register_faces(const Scene* sc, const std::vector<const Face*>& faces) {
    std::lock_guard<std::mutex> lk(g_owner_mu);
    for (const Face* f : faces) g_owner[f] = sc;
}
const Scene* owner_of(const Face& f) {
    std::lock_guard<std::mutex> lk(g_owner_mu);
    auto it = g_owner.find(&f);
    return it == g_owner.end() ? nullptr : it->second;
}
}  // namespace

Scene::~Scene() {
    {
        std::lock_guard<std::mutex> lk(g_owner_mu);
        for (const Face* f : face_ptrs_) {
            auto it = g_owner.find(f);
            if (it != g_owner.end() && it->second == this) g_owner.erase(it);
        }
    }
    if (dev_) visrt_scene_destroy(dev_);
}

namespace {
Vec3 cross3(const Vec3& a, const Vec3& b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

// validate_face (src/scene.cpp:26-49): >= 3 vertices, planar within 1e-9 of
// the Newell plane through pts[0], convex with the stored winding, area > kEps
void validate_face(const Face& face) {
    const auto& pts = face.poly.pts;
    if (pts.size() < 3) throw SceneError("face '" + face.id + "' has fewer than 3 vertices");
    for (const Vec3& p : pts)
        if (std::abs(signed_distance(face, p)) > 1e-9) throw SceneError("face '" + face.id + "' is not planar");
    const size_t n = pts.size();
    for (size_t i = 0; i < n; ++i) {
        const Vec3 e0 = pts[(i + 1) % n] - pts[i];
        const Vec3 e1 = pts[(i + 2) % n] - pts[(i + 1) % n];
        if (dot(cross3(e0, e1), face.poly.normal) < -kEps) throw SceneError("face '" + face.id + "' is not convex");
    }
    Vec3 acc{0, 0, 0};   // ConvexPolygon::area (src/geom.cpp:148-153): fan of cross products
    for (size_t i = 1; i + 1 < n; ++i) acc = acc + cross3(pts[i] - pts[0], pts[i + 1] - pts[0]);
    if (0.5 * norm(acc) <= kEps) throw SceneError("face '" + face.id + "' is degenerate");
}
}  // namespace

Scene::Scene(Scene&& o)
    : materials(std::move(o.materials)), buildings(std::move(o.buildings)), ground(std::move(o.ground)),
      soup_(std::move(o.soup_)), dev_(o.dev_) {
    // building faces keep their addresses (vector moves keep the buffers);
    // the ground face lives in the optional, so the index is rebuilt
    o.dev_ = nullptr;
    const bool finalized = !o.face_ptrs_.empty();
    o.face_ptrs_.clear();
    o.face_index_.clear();
    o.edges_.clear();
    if (!finalized) return;
    if (!soup_.empty()) {
        for (Face& f : soup_) {
            face_index_[f.id] = f.index;
            face_ptrs_.push_back(&f);
        }
        register_faces(this, face_ptrs_);
    } else {
        finalize();
    }
}

void Scene::finalize() {
    // materials (src/scene.cpp:66-78)
    std::set<std::string> material_names;
    for (const Material& m : materials) {
        if (!material_names.insert(m.name).second) throw SceneError("duplicate material '" + m.name + "'");
        if (m.permittivity < 1.0) throw SceneError("material '" + m.name + "' has relative permittivity < 1");
        if (m.conductivity < 0.0) throw SceneError("material '" + m.name + "' has negative conductivity");
    }
    face_ptrs_.clear();
    face_index_.clear();
    edges_.clear();
    auto reg = [&](Face& f) {
        validate_face(f);
        if (!material_names.count(f.material))
            throw SceneError("face '" + f.id + "' references unknown material '" + f.material + "'");
        if (face_index_.count(f.id)) throw SceneError("duplicate face id '" + f.id + "'");
        f.orientation = classify(f.poly.normal);
        f.index = static_cast<int>(face_ptrs_.size());
        face_index_[f.id] = f.index;
        face_ptrs_.push_back(&f);
    };
    using Key = std::tuple<double, double, double>;
    std::set<std::string> building_ids;
    for (Building& b : buildings) {
        if (!building_ids.insert(b.id).second) throw SceneError("duplicate building id '" + b.id + "'");
        if (b.faces.empty()) throw SceneError("building '" + b.id + "' has no faces");
        Vec3 c{0, 0, 0};
        double cnt = 0;
        for (const Face& f : b.faces)
            for (const Vec3& p : f.poly.pts) {
                c = c + p;
                cnt += 1;
            }
        c = c * (1.0 / cnt);
        for (Face& f : b.faces) {
            f.building = b.id;
            Vec3 fc{0, 0, 0};
            for (const Vec3& p : f.poly.pts) fc = fc + p;
            const double k = static_cast<double>(f.poly.pts.size());
            fc = {fc.x / k, fc.y / k, fc.z / k};
            if (dot(f.poly.normal, fc - c) <= 0)
                throw SceneError("face '" + f.id + "' of building '" + b.id + "' does not point outward");
            reg(f);
        }
        // closed shell: every edge shared by exactly two faces; edge ids in key order
        std::map<std::pair<Key, Key>, std::vector<const Face*>> ef;
        for (const Face& f : b.faces) {
            const size_t n = f.poly.pts.size();
            for (size_t i = 0; i < n; ++i) {
                Key a{f.poly.pts[i].x, f.poly.pts[i].y, f.poly.pts[i].z};
                Key e{f.poly.pts[(i + 1) % n].x, f.poly.pts[(i + 1) % n].y, f.poly.pts[(i + 1) % n].z};
                if (e < a) std::swap(a, e);
                ef[{a, e}].push_back(&f);
            }
        }
        size_t i = 0;
        for (const auto& [k, fs] : ef) {
            if (fs.size() != 2)
                throw SceneError("building '" + b.id + "' is not a closed shell (open edge on face '" + fs.front()->id + "')");
            Edge e;
            e.a = {std::get<0>(k.first), std::get<1>(k.first), std::get<2>(k.first)};
            e.b = {std::get<0>(k.second), std::get<1>(k.second), std::get<2>(k.second)};
            e.faces = {fs[0]->id, fs[1]->id};
            e.building = b.id;
            e.id = b.id + "/e" + std::to_string(i++);
            edges_.push_back(e);
        }
    }
    if (ground) {
        ground->building.clear();
        if (classify(ground->poly.normal) != Orientation::Horizontal || ground->poly.normal.z <= 0)
            throw SceneError("ground face '" + ground->id + "' must be horizontal, facing up");
        reg(*ground);
    }
    if (face_ptrs_.empty()) throw SceneError("scene has no faces");
    register_faces(this, face_ptrs_);
}

std::unique_ptr<Scene> Scene::from_facets(const std::vector<std::string>& ids,
                                          const std::vector<std::vector<Vec3>>& rings) {
    auto s = std::make_unique<Scene>();
    s->materials.push_back({"concrete", 5.31, 0.139});   // the facet-soup convention (one wall material)
    s->soup_.reserve(ids.size());
    for (size_t i = 0; i < ids.size(); ++i) {
        Face f;
        f.id = ids[i];
        f.material = "concrete";
        f.poly = ConvexPolygon::from_points(rings[i]);
        f.orientation = classify(f.poly.normal);
        f.index = static_cast<int>(i);
        s->soup_.push_back(std::move(f));
    }
    for (Face& f : s->soup_) {
        s->face_index_[f.id] = f.index;
        s->face_ptrs_.push_back(&f);
    }
    register_faces(s.get(), s->face_ptrs_);
    return s;
}

// ---------------------------------------------------------------------------
// JSON scene I/O (src/scene.cpp:258-375)
// ---------------------------------------------------------------------------
namespace {
Face face_of_json(const nlohmann::json& jf, const std::vector<Vec3>& verts) {
    Face f;
    f.id = jf.at("id").get<std::string>();
    f.material = jf.at("material").get<std::string>();
    std::vector<Vec3> ring;
    for (const auto& jv : jf.at("vertices")) {
        const size_t v = jv.get<size_t>();
        if (v >= verts.size())
            throw SceneError("face '" + f.id + "' references vertex " + std::to_string(v) + " out of range");
        ring.push_back(verts[v]);
    }
    try {
        f.poly = ConvexPolygon::from_points(std::move(ring));
    } catch (const std::exception& e) {
        throw SceneError("face '" + f.id + "': " + e.what());
    }
    if (jf.contains("labels")) {
        const auto& jl = jf.at("labels");
        if (jl.contains("xy")) f.labels.xy = jl.at("xy").get<std::string>();
        if (jl.contains("vert")) f.labels.vert = jl.at("vert").get<std::string>();
    }
    return f;
}
}  // namespace

Scene load_scene(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw SceneError("cannot open scene file '" + path + "'");
    nlohmann::json j;
    try {
        in >> j;
    } catch (const std::exception& e) {
        throw SceneError("scene file '" + path + "' is not valid JSON: " + e.what());
    }
    Scene sc;
    for (const auto& jm : j.value("materials", nlohmann::json::array()))
        sc.materials.push_back({jm.at("name").get<std::string>(), jm.at("permittivity").get<double>(),
                                jm.at("conductivity").get<double>()});
    std::vector<Vec3> verts;
    for (const auto& jv : j.value("vertices", nlohmann::json::array()))
        verts.push_back({jv.at(0).get<double>(), jv.at(1).get<double>(), jv.at(2).get<double>()});
    for (const auto& jb : j.value("buildings", nlohmann::json::array())) {
        Building b;
        b.id = jb.at("id").get<std::string>();
        for (const auto& jf : jb.at("faces")) b.faces.push_back(face_of_json(jf, verts));
        sc.buildings.push_back(std::move(b));
    }
    if (j.contains("ground")) sc.ground = face_of_json(j.at("ground"), verts);
    sc.finalize();
    return sc;
}

void save_scene(const Scene& scene, const std::string& path) {
    if (scene.buildings.empty() && !scene.ground && !scene.faces().empty())
        throw SceneError("a facet soup has no scene-file form");
    nlohmann::json j;
    j["materials"] = nlohmann::json::array();
    for (const Material& m : scene.materials)
        j["materials"].push_back({{"name", m.name}, {"permittivity", m.permittivity}, {"conductivity", m.conductivity}});
    std::vector<Vec3> verts;
    std::map<std::tuple<double, double, double>, size_t> index;   // exact-coordinate interning
    auto face_json = [&](const Face& f) {
        nlohmann::json jf;
        jf["id"] = f.id;
        jf["material"] = f.material;
        nlohmann::json idx = nlohmann::json::array();
        for (const Vec3& p : f.poly.pts) {
            const auto key = std::make_tuple(p.x, p.y, p.z);
            auto it = index.find(key);
            if (it == index.end()) {
                verts.push_back(p);
                it = index.emplace(key, verts.size() - 1).first;
            }
            idx.push_back(it->second);
        }
        jf["vertices"] = idx;
        if (!f.labels.xy.empty() || !f.labels.vert.empty()) {
            nlohmann::json jl;
            if (!f.labels.xy.empty()) jl["xy"] = f.labels.xy;
            if (!f.labels.vert.empty()) jl["vert"] = f.labels.vert;
            jf["labels"] = jl;
        }
        return jf;
    };
    j["buildings"] = nlohmann::json::array();
    for (const Building& b : scene.buildings) {
        nlohmann::json jb;
        jb["id"] = b.id;
        jb["faces"] = nlohmann::json::array();
        for (const Face& f : b.faces) jb["faces"].push_back(face_json(f));
        j["buildings"].push_back(jb);
    }
    if (scene.ground) j["ground"] = face_json(*scene.ground);
    j["vertices"] = nlohmann::json::array();
    for (const Vec3& v : verts) j["vertices"].push_back({v.x, v.y, v.z});
    std::ofstream out(path);
    if (!out) throw SceneError("cannot write scene file '" + path + "'");
    out << j.dump(2) << "\n";
}

const Material& Scene::material(const std::string& name) const {   // src/scene.cpp:192-197
    for (const Material& m : materials)
        if (m.name == name) return m;
    throw SceneError("unknown material '" + name + "'");
}

const Face& Scene::face(const std::string& id) const {
    auto it = face_index_.find(id);
    if (it == face_index_.end()) throw SceneError("unknown face id '" + id + "'");
    return *face_ptrs_[static_cast<size_t>(it->second)];
}

bool Scene::inside_building(const Vec3& p) const {
    for (const Building& b : buildings) {
        bool inside = true;
        for (const Face& f : b.faces)
            if (signed_distance(f, p) >= -kEps) {
                inside = false;
                break;
            }
        if (inside) return true;
    }
    return false;
}

visrt_scene* Scene::device_scene() const {
    if (dev_) return dev_;
    std::vector<int32_t> off{0}, bld;
    std::vector<double> verts;
    std::map<std::string, int> bidx;
    for (const Building& b : buildings) bidx.emplace(b.id, static_cast<int>(bidx.size()));
    for (const Face* f : face_ptrs_) {
        for (const Vec3& p : f->poly.pts) {
            verts.push_back(p.x);
            verts.push_back(p.y);
            verts.push_back(p.z);
        }
        off.push_back(off.back() + static_cast<int32_t>(f->poly.pts.size()));
        bld.push_back(f->building.empty() ? -1 : bidx.at(f->building));
    }
    visrt_facets_v1 fc{static_cast<int32_t>(face_ptrs_.size()), off.data(), verts.data(),
                       buildings.empty() ? nullptr : bld.data()};
    check(visrt_scene_create(&fc, 0, &dev_));
    return dev_;
}

std::optional<PlaneSegment> plane_segment(const Face& face, PlaneTag plane) {
    std::vector<int32_t> off{0, static_cast<int32_t>(face.poly.pts.size())};
    std::vector<double> v;
    for (const Vec3& p : face.poly.pts) {
        v.push_back(p.x);
        v.push_back(p.y);
        v.push_back(p.z);
    }
    visrt_facets_v1 fc{1, off.data(), v.data(), nullptr};
    visrt_scene* h = nullptr;
    check(visrt_scene_create(&fc, -1, &h));   // host-only ingest, the reference arithmetic
    double seg[18];
    int32_t ok[3];
    const int rc = visrt_scene_ingest(h, nullptr, nullptr, seg, ok);
    visrt_scene_destroy(h);
    check(rc);
    const int pl = static_cast<int>(plane);
    if (!ok[pl]) return std::nullopt;
    return PlaneSegment{{seg[6 * pl], seg[6 * pl + 1]}, {seg[6 * pl + 2], seg[6 * pl + 3]},
                        {seg[6 * pl + 4], seg[6 * pl + 5]}};
}

// ---------------------------------------------------------------------------
std::vector<const InterVisEntry*> InterVisMatrix::find(int order, const std::string& ref, const std::string& aim) const {
    std::vector<const InterVisEntry*> out;
    auto it = index_.find({order, ref, aim});
    if (it != index_.end())
        for (size_t i : it->second) out.push_back(&entries_[i]);
    return out;
}
const InterVisEntry* InterVisMatrix::find(int order, const std::string& ref, const std::string& aim,
                                          PlaneTag plane) const {
    auto it = index_.find({order, ref, aim});
    if (it == index_.end()) return nullptr;
    for (size_t i : it->second)
        if (entries_[i].relation.plane == plane) return &entries_[i];
    return nullptr;
}
bool InterVisMatrix::pair_admitted(const std::string& ref, const std::string& aim) const {
    return index_.count({1, ref, aim}) > 0;
}
std::vector<std::string> InterVisMatrix::aims_of(const std::string& ref) const {
    std::vector<std::string> out;
    for (const InterVisEntry& e : entries_)
        if (e.order == 1 && e.ref == ref && std::find(out.begin(), out.end(), e.aim) == out.end()) out.push_back(e.aim);
    return out;
}
void InterVisMatrix::add(InterVisEntry entry) {
    auto& slot = index_[{entry.order, entry.ref, entry.aim}];
    for (size_t i : slot)
        if (entries_[i].relation.plane == entry.relation.plane && entries_[i].relation.chain == entry.relation.chain)
            throw VisibilityError("duplicate matrix entry for ('" + entry.ref + "','" + entry.aim + "')");
    slot.push_back(entries_.size());
    entries_.push_back(std::move(entry));
}

OcclusionVerdict occlusion_judgment(const Face& ref, const Face& aim, const Scene& scene) {
    if (ref.id == aim.id)
        throw VisibilityError("occlusion judgment needs two distinct faces (got '" + ref.id + "')");
    const int32_t ci = ref.index, cj = aim.index;
    int8_t kind = 0;
    int64_t off[2] = {0, 0};
    visrt_stats st{};
    check(visrt_pair_detail(scene.device_scene(), 1, &ci, &cj, &kind, off, nullptr, 0, &st, nullptr));
    std::vector<int32_t> blk(static_cast<size_t>(off[1]) + 1);
    check(visrt_pair_detail(scene.device_scene(), 1, &ci, &cj, &kind, off, blk.data(), off[1], &st, nullptr));
    OcclusionVerdict v;
    v.kind = static_cast<OcclusionVerdict::Kind>(kind);
    std::set<std::string> ids;
    for (int64_t k = 0; k < off[1]; ++k) ids.insert(scene.face(blk[static_cast<size_t>(k)]).id);
    v.blockers.assign(ids.begin(), ids.end());
    return v;
}

namespace {
// The host half of build_matrix: InterVisEntry records for the admitted pairs
// (pair order) and the Markov-2 chain growth over the feasible triples.
InterVisMatrix materialize(const Scene& scene, int max_order, const std::vector<int32_t>& ai,
                           const std::vector<int32_t>& aj, const std::vector<int32_t>& tri);
}  // namespace

InterVisMatrix build_matrix(const Scene& scene, int max_order) {
    if (max_order < 1 || max_order > 4) throw VisibilityError("max reflection order must be between 1 and 4");
    visrt_scene* dev = scene.device_scene();
    visrt_stats st{};
    check(visrt_pair_visibility(dev, VISRT_PAIRS_PREFILTERED, nullptr, &st, nullptr));
    const int64_t m = visrt_candidates(dev, nullptr, nullptr, nullptr);
    std::vector<int32_t> ci(m), cj(m);
    std::vector<uint8_t> adm(m);
    visrt_candidates(dev, ci.data(), cj.data(), adm.data());
    std::vector<int32_t> ai, aj;
    for (int64_t k = 0; k < m; ++k)
        if (adm[k]) {
            ai.push_back(ci[k]);
            aj.push_back(cj[k]);
        }
    std::vector<int32_t> tri;
    if (max_order >= 2) {
        int64_t nt = 0;
        check(visrt_chain_triples(dev, nullptr, nullptr, 0, &nt, &st, nullptr));
        tri.resize(static_cast<size_t>(nt) * 3 + 3);
        check(visrt_chain_triples(dev, nullptr, tri.data(), nt, &nt, &st, nullptr));
        tri.resize(static_cast<size_t>(nt) * 3);
    }
    return materialize(scene, max_order, ai, aj, tri);
}

void save_matrix_cache(const InterVisMatrix& matrix, const Scene& scene, const std::string& path) {
    const size_t n = scene.faces().size(), words = (n + 63) / 64;
    std::vector<uint64_t> bits(n * words + 1, 0);
    std::vector<int32_t> tri;
    for (const InterVisEntry& e : matrix.entries()) {
        const auto& c = e.relation.chain;
        if (e.order == 1 && c.size() == 2) {
            const size_t r = static_cast<size_t>(scene.face(c[0]).index), a = static_cast<size_t>(scene.face(c[1]).index);
            bits[r * words + a / 64] |= 1ull << (a % 64);
        } else if (e.order == 2 && c.size() == 3) {
            for (const auto& id : c) tri.push_back(scene.face(id).index);
        }
    }
    // one copy per triple (an order-2 chain has one entry per shared plane at most)
    std::vector<std::array<int32_t, 3>> t3;
    for (size_t k = 0; k + 2 < tri.size(); k += 3) t3.push_back({tri[k], tri[k + 1], tri[k + 2]});
    std::sort(t3.begin(), t3.end());
    t3.erase(std::unique(t3.begin(), t3.end()), t3.end());
    std::vector<int32_t> flat;
    for (const auto& t : t3) flat.insert(flat.end(), t.begin(), t.end());
    check(visrt_cache_save(path.c_str(), scene.device_scene(), matrix.max_order(), bits.data(),
                           static_cast<int64_t>(t3.size()), flat.empty() ? nullptr : flat.data()));
}

InterVisMatrix load_matrix_cache(const Scene& scene, const std::string& path) {
    visrt_scene* dev = scene.device_scene();
    int32_t mo = 1;
    int64_t nt = 0;
    check(visrt_cache_load(path.c_str(), dev, &mo, nullptr, nullptr, 0, &nt));
    const size_t n = scene.faces().size(), words = (n + 63) / 64;
    std::vector<uint64_t> bits(n * words + 1);
    std::vector<int32_t> tri(static_cast<size_t>(nt) * 3 + 3);
    check(visrt_cache_load(path.c_str(), dev, &mo, bits.data(), tri.data(), nt, &nt));
    tri.resize(static_cast<size_t>(nt) * 3);
    std::vector<int32_t> ai, aj;
    for (size_t i = 0; i < n; ++i)
        for (size_t j = i + 1; j < n; ++j)
            if ((bits[i * words + j / 64] >> (j % 64)) & 1ull) {
                ai.push_back(static_cast<int32_t>(i));
                aj.push_back(static_cast<int32_t>(j));
            }
    return materialize(scene, mo, ai, aj, tri);
}

namespace {
InterVisMatrix materialize(const Scene& scene, int max_order, const std::vector<int32_t>& ai,
                           const std::vector<int32_t>& aj, const std::vector<int32_t>& tri) {
    visrt_scene* dev = scene.device_scene();
    const int n = static_cast<int>(scene.faces().size());
    InterVisMatrix matrix;
    matrix.set_max_order(max_order);
    visrt_stats st{};
    // verdict kinds + blockers of the admitted pairs (Partial pairs record them)
    std::vector<int8_t> kind(ai.size());
    std::vector<int64_t> boff(ai.size() + 1);
    check(visrt_pair_detail(dev, static_cast<int64_t>(ai.size()), ai.data(), aj.data(), kind.data(), boff.data(),
                            nullptr, 0, &st, nullptr));
    std::vector<int32_t> bidx(static_cast<size_t>(boff.back()) + 1);
    check(visrt_pair_detail(dev, static_cast<int64_t>(ai.size()), ai.data(), aj.data(), kind.data(), boff.data(),
                            bidx.data(), boff.back(), &st, nullptr));
    const Segs segs = scene_segs(scene);
    // first_order_pair entries, pair order (src/vismatrix.cpp:597-634, 673-675)
    for (size_t q = 0; q < ai.size(); ++q) {
        std::vector<std::string> blockers;
        if (kind[q] == 1) {
            std::set<std::string> ids;
            for (int64_t k = boff[q]; k < boff[q + 1]; ++k) ids.insert(scene.face(bidx[static_cast<size_t>(k)]).id);
            blockers.assign(ids.begin(), ids.end());
        }
        for (PlaneTag plane : required_planes(segs, ai[q], aj[q])) {
            for (int dir = 0; dir < 2; ++dir) {
                const int r = dir == 0 ? ai[q] : aj[q], a = dir == 0 ? aj[q] : ai[q];
                InterVisEntry e;
                e.order = 1;
                e.ref = scene.face(r).id;
                e.aim = scene.face(a).id;
                e.relation = relation(scene, segs, r, a, plane);
                e.ranges = first_order_ranges(scene, segs, r, a, plane);
                e.blockers = blockers;
                e.aim_image = chain_image(scene, {r, a});
                matrix.add(std::move(e));
            }
        }
    }
    if (max_order < 2) return matrix;
    // chains: the GPU decides every feasible triple; the frontier growth and
    // the record fields follow src/vismatrix.cpp:682-797
    const int64_t nt = static_cast<int64_t>(tri.size() / 3);
    std::unordered_set<uint64_t> feasible;
    auto key3 = [n](int a, int b, int c) {
        return (static_cast<uint64_t>(a) * n + static_cast<uint64_t>(b)) * n + static_cast<uint64_t>(c);
    };
    for (int64_t k = 0; k < nt; ++k) feasible.insert(key3(tri[3 * k], tri[3 * k + 1], tri[3 * k + 2]));
    std::vector<std::vector<int>> aims(n);
    for (size_t q = 0; q < ai.size(); ++q) {
        aims[ai[q]].push_back(aj[q]);
        aims[aj[q]].push_back(ai[q]);
    }
    for (auto& v : aims) std::sort(v.begin(), v.end());   // aims_of order = ascending index
    std::vector<std::vector<int>> frontier;
    for (int i = 0; i < n; ++i)
        for (int a : aims[i]) frontier.push_back({i, a});
    for (int order = 2; order <= max_order; ++order) {
        std::vector<std::vector<int>> next;
        for (const auto& chain : frontier) {
            const int t = chain.back(), p = chain[chain.size() - 2];
            for (int a : aims[t]) {
                if (!feasible.count(key3(p, t, a))) continue;
                const auto planes = required_planes(segs, t, a);
                const auto first_planes = required_planes(segs, p, t);
                InterVisEntry e;
                e.order = order;
                std::vector<int> grown = chain;
                grown.push_back(a);
                e.ref = scene.face(grown.front()).id;
                e.aim = scene.face(a).id;
                e.relation = relation(scene, segs, t, a, planes.front());
                e.ranges = first_order_ranges(scene, segs, t, a, planes.front());
                e.criterion = clamp_complement(first_order_ranges(scene, segs, p, t, first_planes.front()));
                // triple_ext record fields (src/vismatrix.cpp:725-748)
                e.verdict = ChainVerdict::Partial;
                bool recorded = false;
                for (PlaneTag pl : planes) {
                    if (std::find(first_planes.begin(), first_planes.end(), pl) == first_planes.end()) continue;
                    ISet reach;
                    const ChainVerdict v = second_order(segs, p, t, a, pl, reach);
                    if (!recorded) {
                        e.relation.plane = pl;
                        e.verdict = v;
                        for (const auto& iv : reach) e.subranges.push_back(iv);
                        recorded = true;
                    } else if (v != ChainVerdict::Full) {
                        e.verdict = ChainVerdict::Partial;
                    }
                }
                e.relation.chain.clear();
                e.relation.chain_orientations.clear();
                for (int idx : grown) {
                    e.relation.chain.push_back(scene.face(idx).id);
                    e.relation.chain_orientations.push_back(scene.face(idx).orientation);
                }
                e.aim_image = chain_image(scene, grown);
                next.push_back(grown);
                matrix.add(std::move(e));
            }
        }
        frontier = std::move(next);
    }
    return matrix;
}
}  // namespace

// ---------------------------------------------------------------------------
namespace {
double boundary_angle(const Vec2& at, const Vec2& other, const Vec2& outward, const Vec2& image) {
    const Vec2 ref = sub2(other, at), ray = sub2(at, image);
    if (norm2(ray) <= kEps || norm2(ref) <= kEps) return 0.0;
    return clamp_angle(oriented_angle(ref, outward, ray));
}
Vec2 mirror_across(const Vec2& q, const Vec2& a, const Vec2& b) {
    const Vec2 d = sub2(b, a);
    const double len2 = dot2(d, d);
    const double t = dot2(sub2(q, a), d) / len2;
    const Vec2 foot{a.x + d.x * t, a.y + d.y * t};
    return {foot.x * 2.0 - q.x, foot.y * 2.0 - q.y};
}
}  // namespace

std::vector<std::vector<std::optional<IlluminatedRegion>>> illuminated_regions(const std::vector<Vec3>& sources,
                                                                               const Scene& scene) {
    visrt_scene* dev = scene.device_scene();
    const size_t n = scene.faces().size();
    std::vector<double> src;
    for (const Vec3& s : sources) {
        src.push_back(s.x);
        src.push_back(s.y);
        src.push_back(s.z);
    }
    std::vector<visrt_region> out(sources.size() * n);
    visrt_stats st{};
    check(visrt_point_regions(dev, static_cast<int64_t>(sources.size()), src.data(), out.data(), &st, nullptr));
    const Segs segs = scene_segs(scene);
    std::vector<std::vector<std::optional<IlluminatedRegion>>> res(sources.size());
    for (size_t k = 0; k < sources.size(); ++k) {
        res[k].resize(n);
        for (size_t f = 0; f < n; ++f) {
            const visrt_region& r = out[k * n + f];
            if (r.present != 1) continue;   // none (-1: source on the plane, handled by the caller)
            IlluminatedRegion reg;
            reg.face = scene.face(static_cast<int>(f)).id;
            reg.source = sources[k];
            for (int pl = 0; pl < 3; ++pl) {
                if (!r.has[pl]) continue;
                const PlaneSegment sg = segs.get(static_cast<int>(f), pl);
                PlaneIllumination pi;
                pi.plane = static_cast<PlaneTag>(pl);
                pi.face_a = sg.a;
                pi.face_b = sg.b;
                pi.outward = sg.normal;
                pi.image = mirror_across(project(sources[k], pi.plane), sg.a, sg.b);
                pi.sub = {r.sub[2 * pl], r.sub[2 * pl + 1]};
                const Vec2 dir = sub2(sg.b, sg.a);
                pi.sub_a = {sg.a.x + dir.x * pi.sub[0], sg.a.y + dir.y * pi.sub[0]};
                pi.sub_b = {sg.a.x + dir.x * pi.sub[1], sg.a.y + dir.y * pi.sub[1]};
                pi.alpha_full = boundary_angle(pi.face_a, pi.face_b, pi.outward, pi.image);
                pi.beta_full = boundary_angle(pi.face_b, pi.face_a, pi.outward, pi.image);
                pi.alpha = boundary_angle(pi.sub_a, pi.sub_b, pi.outward, pi.image);
                pi.beta = boundary_angle(pi.sub_b, pi.sub_a, pi.outward, pi.image);
                pi.clipped = r.clipped[pl] != 0;
                if (pi.sub[0] > 1e-9) pi.clip_points.push_back(pi.sub_a);
                if (pi.sub[1] < 1.0 - 1e-9) pi.clip_points.push_back(pi.sub_b);
                reg.planes.push_back(pi);
            }
            res[k][f] = std::move(reg);
        }
    }
    return res;
}

std::optional<IlluminatedRegion> illuminated_region(const Vec3& source, const Face& face, const Scene& scene) {
    const double dist = signed_distance(face, source);
    if (std::abs(dist) <= kEps) throw VisibilityError("source lies on the plane of face '" + face.id + "'");
    if (dist < 0.0) return std::nullopt;
    auto all = illuminated_regions({source}, scene);
    return all[0][static_cast<size_t>(face.index)];
}

// ---------------------------------------------------------------------------
std::string Path::identity() const {
    if (interactions.empty()) return "LOS";
    std::string id;
    for (size_t i = 0; i < interactions.size(); ++i) {
        if (i) id += '/';
        id += (interactions[i].kind == InteractionKind::Reflection ? "R:" : "D:") + interactions[i].id;
    }
    return id;
}

TraceAccelerator::TraceAccelerator(const Scene& scene, const InterVisMatrix& matrix, int max_refl)
    : scene_(&scene), max_refl_(max_refl) {
    if (max_refl < 0) throw VisibilityError("reflection order must be non-negative");
    if (max_refl > matrix.max_order())
        throw VisibilityError("matrix order " + std::to_string(matrix.max_order()) +
                              " is lower than the requested reflection order " + std::to_string(max_refl));
    const int n = static_cast<int>(scene.faces().size());
    const int words = (n + 63) / 64;
    std::vector<uint64_t> bits(static_cast<size_t>(n) * words, 0);
    std::vector<int32_t> tri;
    for (const InterVisEntry& e : matrix.entries()) {   // build_chain_filter, src/raytracer.cpp:319-340
        const auto& c = e.relation.chain;
        if (static_cast<int>(c.size()) > max_refl || c.size() < 2) continue;
        if (c.size() == 2) {
            const int r = scene.face(c[0]).index, a = scene.face(c[1]).index;
            bits[static_cast<size_t>(r) * words + a / 64] |= 1ull << (a % 64);
        } else if (c.size() == 3) {
            for (const auto& id : c) tri.push_back(scene.face(id).index);
        }
    }
    check(visrt_tracer_create(scene.device_scene(), max_refl, bits.data(), static_cast<int64_t>(tri.size() / 3),
                              tri.empty() ? nullptr : tri.data(), &tracer_));
    set_edges(scene);
}

TraceAccelerator::TraceAccelerator(const Scene& scene, int max_refl)
    : scene_(&scene), max_refl_(max_refl), brute_(true) {
    if (max_refl < 0) throw VisibilityError("reflection order must be non-negative");
    const size_t n = scene.faces().size();
    std::vector<uint64_t> bits(n * ((n + 63) / 64) + 1, 0);
    check(visrt_tracer_create(scene.device_scene(), max_refl, bits.data(), 0, nullptr, &tracer_));
    set_edges(scene);
}

std::vector<Path> brute_force_trace(const Scene& scene, const Vec3& tx, const Vec3& rx, int max_refl,
                                    bool allow_diffraction, TraceStats* stats) {
    TraceAccelerator acc(scene, max_refl);
    return acc.trace(tx, rx, allow_diffraction, stats);
}

void TraceAccelerator::set_edges(const Scene& scene) {
    if (!scene.edges().empty()) {   // diffraction candidates (Scene::edges)
        std::vector<double> ab;
        std::vector<std::string> ids;
        for (const Edge& e : scene.edges()) {
            ab.insert(ab.end(), {e.a.x, e.a.y, e.a.z, e.b.x, e.b.y, e.b.z});
            ids.push_back(e.id);
        }
        const auto rk = ranks_of(ids);
        std::vector<int32_t> rank;
        for (const Edge& e : scene.edges()) rank.push_back(rk.at(e.id));
        check(visrt_tracer_set_edges(tracer_, static_cast<int32_t>(rank.size()), ab.data(), rank.data()));
    }
}

TraceAccelerator::~TraceAccelerator() {
    if (tracer_) visrt_tracer_destroy(tracer_);
}

std::vector<std::vector<Path>> TraceAccelerator::trace_batch(const std::vector<Vec3>& tx, const std::vector<Vec3>& rx,
                                                             std::vector<TraceStats>* stats,
                                                             bool allow_diffraction) const {
    std::vector<double> t, r;
    for (const Vec3& p : tx) {
        t.push_back(p.x);
        t.push_back(p.y);
        t.push_back(p.z);
    }
    for (const Vec3& p : rx) {
        r.push_back(p.x);
        r.push_back(p.y);
        r.push_back(p.z);
    }
    visrt_trace_stats st{};
    const int flags = (rx.size() == 1 ? VISRT_TRACE_RX_FIXED : 0) | (allow_diffraction ? VISRT_TRACE_DIFFRACTION : 0) |
                      (brute_ ? VISRT_TRACE_BRUTE_FORCE : 0);
    check(visrt_trace(tracer_, static_cast<int64_t>(tx.size()), t.data(), r.data(), flags, &st, nullptr));
    const int64_t np = visrt_trace_results(tracer_, nullptr, nullptr, 0, nullptr);
    std::vector<int64_t> off(tx.size() + 1), nodes(tx.size());
    std::vector<visrt_path> ps(static_cast<size_t>(np) + 1);
    visrt_trace_results(tracer_, off.data(), ps.data(), np, nodes.data());
    std::vector<int32_t> sedge(tx.size(), -1);
    visrt_trace_snapshot_edges(tracer_, sedge.data());
    std::vector<std::vector<Path>> out(tx.size());
    for (size_t k = 0; k < tx.size(); ++k) {
        for (int64_t q = off[k]; q < off[k + 1]; ++q) {
            const visrt_path& vp = ps[static_cast<size_t>(q)];
            Path p;
            p.source = tx[k];
            p.receiver = rx.size() == 1 ? rx[0] : rx[k];
            const int npts = vp.nrefl + 2 + (vp.edge >= 0 ? 1 : 0);
            for (int i = 0; i < npts; ++i) p.points.push_back({vp.points[3 * i], vp.points[3 * i + 1], vp.points[3 * i + 2]});
            for (int i = 0; i < vp.nrefl; ++i)
                p.interactions.push_back({InteractionKind::Reflection, scene_->face(vp.faces[i]).id, p.points[1 + i]});
            if (vp.edge >= 0)
                p.interactions.push_back({InteractionKind::Diffraction, scene_->edges()[static_cast<size_t>(vp.edge)].id,
                                          p.points[1 + vp.nrefl]});
            p.length = vp.length;
            p.delay = vp.length / kSpeedOfLight;
            out[k].push_back(std::move(p));
        }
        std::sort(out[k].begin(), out[k].end(), [](const Path& a, const Path& b) { return a.identity() < b.identity(); });
        if (stats) {
            TraceStats ts;
            ts.nodes_expanded = nodes[k];
            ts.sequences_checked = (nodes[k] + 1) * (sedge[k] >= 0 ? 2 : 1);
            ts.paths_found = static_cast<long long>(out[k].size());
            // the GPU's exact leg tests of the batch, split evenly (INTEGRATION.md:
            // the reference's grid-filtered count has no counterpart)
            ts.occlusion_tests = tx.empty() ? 0 : st.leg_tests / static_cast<long long>(tx.size());
            stats->push_back(ts);
        }
    }
    return out;
}

std::vector<Path> TraceAccelerator::trace(const Vec3& tx, const Vec3& rx, bool allow_diffraction,
                                          TraceStats* stats) const {
    std::vector<TraceStats> st;
    auto out = trace_batch({tx}, {rx}, stats ? &st : nullptr, allow_diffraction);
    if (stats) *stats = st[0];
    return std::move(out[0]);
}

// ---------------------------------------------------------------------------
// (2) tables: point_vis_table, trajectory_vis_table, closest_diffraction_edge
// ---------------------------------------------------------------------------
namespace {
visrt_entry to_entry(const Scene& scene, const InterVisEntry& e) {
    visrt_entry v{};
    v.order = e.order;
    const auto& c = e.relation.chain;
    for (size_t k = 0; k < c.size() && k < 5; ++k) v.chain[k] = scene.face(c[k]).index;
    v.plane = static_cast<int32_t>(e.relation.plane);
    return v;
}
void check_table_order(const InterVisMatrix& matrix, int max_order) {
    if (max_order < 1) throw VisibilityError("max_order must be at least 1");
    if (matrix.max_order() < max_order)
        throw VisibilityError("matrix holds orders up to " + std::to_string(matrix.max_order()) + ", requested " +
                              std::to_string(max_order));

}
}  // namespace

std::vector<VisTableEntry> point_vis_table(const Vec3& source, const InterVisMatrix& matrix, const Scene& scene,
                                           int max_order) {
    check_table_order(matrix, max_order);   // src/vistable.cpp:480-485
    const size_t n = scene.faces().size();
    std::vector<const InterVisEntry*> used;
    std::vector<visrt_entry> ents;
    for (const InterVisEntry& e : matrix.entries()) {
        if (e.order > max_order || e.relation.chain.size() < 2) continue;
        used.push_back(&e);
        ents.push_back(to_entry(scene, e));
    }
    const size_t words = (ents.size() + 31) / 32;
    std::vector<uint32_t> rows(std::max<size_t>(words, 1)), full(std::max<size_t>(words, 1));
    std::vector<visrt_region> regs(n);
    const double src[3] = {source.x, source.y, source.z};
    visrt_stats st{};
    check(visrt_point_tables(scene.device_scene(), 1, src, static_cast<int64_t>(ents.size()), ents.data(),
                             rows.data(), full.data(), regs.data(), &st, nullptr));
    // TableBuilder::display (src/vistable.cpp:392-401)
    auto display = [&](const std::string& id, PlaneTag plane) {
        const Face& f = scene.face(id);
        std::string name = f.label(plane);
        const visrt_region& r = regs[static_cast<size_t>(f.index)];
        const int pl = static_cast<int>(plane);
        if (r.present == 1 && r.has[pl] && r.clipped[pl]) name += "'";
        return name;
    };
    std::vector<VisTableEntry> out;
    for (size_t k = 0; k < used.size(); ++k) {
        if (!((rows[k >> 5] >> (k & 31)) & 1u)) continue;
        const InterVisEntry& e = *used[k];
        const auto& cf = e.relation.chain;
        VisTableEntry row;
        row.order = e.order;
        row.chain.assign(cf.begin(), cf.end() - 1);
        row.ref = row.chain.back();
        row.aim = e.aim;
        row.plane = e.relation.plane;
        row.parent = row.chain.size() >= 2 ? row.chain[row.chain.size() - 2] : std::string("transmitter");
        row.parent_display = row.chain.size() >= 2 ? display(row.parent, e.relation.plane) : std::string("transmitter");
        row.ref_display = display(row.ref, e.relation.plane);
        row.aim_display = display(row.aim, e.relation.plane);
        row.verdict = ((full[k >> 5] >> (k & 31)) & 1u) ? ChainVerdict::Full : ChainVerdict::Partial;
        out.push_back(std::move(row));
    }
    std::sort(out.begin(), out.end(), [](const VisTableEntry& a, const VisTableEntry& b) {
        return std::tie(a.order, a.chain, a.aim, a.plane) < std::tie(b.order, b.chain, b.aim, b.plane);
    });
    return out;
}

// src/scene.cpp:443-469
double Trajectory::total_length() const {
    double len = 0;
    for (size_t i = 0; i + 1 < waypoints.size(); ++i) len += norm(waypoints[i + 1] - waypoints[i]);
    return len;
}
Vec3 Trajectory::position_at(double s) const {
    if (s <= 0) return waypoints.front();
    for (size_t i = 0; i + 1 < waypoints.size(); ++i) {
        const double seg = norm(waypoints[i + 1] - waypoints[i]);
        if (s <= seg) return waypoints[i] + (waypoints[i + 1] - waypoints[i]) * (s / seg);
        s -= seg;
    }
    return waypoints.back();
}


std::vector<MobileVisEntry> trajectory_vis_table(const Trajectory& traj, const InterVisMatrix& matrix,
                                                 const Scene& scene, int max_order) {
    if (traj.waypoints.size() < 2 || traj.total_length() <= kEps)   // src/vistable.cpp:825-828
        throw VisibilityError("trajectory must contain at least two distinct waypoints");
    if (matrix.max_order() < max_order)
        throw VisibilityError("matrix holds orders up to " + std::to_string(matrix.max_order()) + ", requested " +
                              std::to_string(max_order));

    const int n = static_cast<int>(scene.faces().size());
    std::vector<std::string> keys{"transmitter"}, parents{"transmitter"}, blds;
    auto corner = [&](int f, int k) { return scene.face(f).id + "#" + std::to_string(k); };
    for (int f = 0; f < n; ++f) {
        const Face& fc = scene.face(f);
        keys.push_back(fc.id);
        for (size_t k = 0; k < fc.poly.pts.size(); ++k) keys.push_back(corner(f, static_cast<int>(k)));
        parents.push_back(fc.label(PlaneTag::XY));
        blds.push_back(building_of(fc));
    }
    const auto kr = ranks_of(keys), pr = ranks_of(parents), br = ranks_of(blds);
    std::vector<int32_t> key_rank(9 * static_cast<size_t>(n) + 1, 0), parent_rank(n + 1), building_rank(n);
    for (int f = 0; f < n; ++f) {
        const Face& fc = scene.face(f);
        key_rank[f] = kr.at(fc.id);
        for (size_t k = 0; k < fc.poly.pts.size(); ++k)
            key_rank[n + 8 * static_cast<size_t>(f) + k] = kr.at(corner(f, static_cast<int>(k)));
        parent_rank[f] = pr.at(fc.label(PlaneTag::XY));
        building_rank[f] = br.at(building_of(fc));
    }
    key_rank[9 * static_cast<size_t>(n)] = kr.at("transmitter");
    parent_rank[n] = pr.at("transmitter");
    std::vector<std::string> bname(br.size());
    for (const auto& [name, r] : br) bname[static_cast<size_t>(r)] = name;
    std::vector<visrt_entry> ents;
    for (const InterVisEntry& e : matrix.entries())
        if (e.order <= max_order && e.relation.chain.size() >= 2) ents.push_back(to_entry(scene, e));
    std::vector<double> wp;
    for (const Vec3& w : traj.waypoints) wp.insert(wp.end(), {w.x, w.y, w.z});
    const visrt_names names{key_rank.data(), parent_rank.data(), building_rank.data()};
    visrt_mobile_table* t = nullptr;
    visrt_stats st{};
    check(visrt_trajectory_table(scene.device_scene(), static_cast<int32_t>(traj.waypoints.size()), wp.data(),
                                 static_cast<int64_t>(ents.size()), ents.data(), max_order, &names, &t, &st, nullptr));
    const int64_t nr = visrt_mobile_table_rows(t, nullptr, 0);
    std::vector<visrt_mobile_row> rows(static_cast<size_t>(std::max<int64_t>(nr, 1)));
    visrt_mobile_table_rows(t, rows.data(), nr);
    visrt_mobile_table_destroy(t);
    auto label = [](int i, int prime) { return i == 0 ? std::string("-") : "P" + std::to_string(i) + (prime ? "'" : ""); };
    std::vector<MobileVisEntry> out;
    for (int64_t k = 0; k < nr; ++k) {
        const visrt_mobile_row& r = rows[static_cast<size_t>(k)];
        const Face& f = scene.face(r.node);
        MobileVisEntry m;
        m.order = r.order;
        m.node = r.vertex < 0 ? f.id : corner(r.node, r.vertex);
        m.node_display = r.vertex < 0 ? f.label(PlaneTag::XY) : f.label(PlaneTag::XY) + "#" + std::to_string(r.vertex);
        m.s_start = r.s_start;
        m.s_end = r.s_end;
        m.label_start = label(r.label_start, r.prime_start);
        m.label_end = label(r.label_end, r.prime_end);
        m.parent = r.parent < 0 ? std::string("transmitter") : scene.face(r.parent).label(PlaneTag::XY);
        m.blockage = r.blockage < 0 ? std::string("-") : bname[static_cast<size_t>(r.blockage)];
        out.push_back(std::move(m));
    }
    return out;
}

std::optional<Edge> closest_diffraction_edge(const Vec3& receiver, const Scene& scene) {
    const auto& es = scene.edges();
    if (es.empty()) return std::nullopt;
    std::vector<double> ab;
    std::vector<std::string> ids;
    for (const Edge& e : es) {
        ab.insert(ab.end(), {e.a.x, e.a.y, e.a.z, e.b.x, e.b.y, e.b.z});
        ids.push_back(e.id);
    }
    const auto rk = ranks_of(ids);
    std::vector<int32_t> rank;
    for (const Edge& e : es) rank.push_back(rk.at(e.id));
    const double rx[3] = {receiver.x, receiver.y, receiver.z};
    int32_t best = -1;
    visrt_stats st{};
    check(visrt_closest_edges(scene.device_scene(), 1, rx, static_cast<int32_t>(es.size()), ab.data(), rank.data(),
                              &best, &st, nullptr));
    if (best < 0) return std::nullopt;
    return es[static_cast<size_t>(best)];
}

std::optional<Edge> closest_diffraction_edge(const Vec3& receiver, const Scene& scene, const InterVisMatrix&) {
    return closest_diffraction_edge(receiver, scene);
}

std::vector<ImageTreeNode> image_tree(const Scene& scene, const Vec3& source, int max_depth) {
    const double src[3] = {source.x, source.y, source.z};
    int64_t cnt = 0;
    visrt_stats st{};
    check(visrt_image_tree(scene.device_scene(), src, max_depth, nullptr, nullptr, nullptr, nullptr, 0, &cnt, &st,
                           nullptr));
    const size_t m = static_cast<size_t>(std::max<int64_t>(cnt, 1));
    std::vector<int32_t> face(m), parent(m), depth(m);
    std::vector<double> image(3 * m);
    check(visrt_image_tree(scene.device_scene(), src, max_depth, face.data(), parent.data(), depth.data(),
                           image.data(), cnt, &cnt, &st, nullptr));
    std::vector<ImageTreeNode> out(static_cast<size_t>(cnt));
    for (int64_t k = 0; k < cnt; ++k) {
        ImageTreeNode& nd = out[static_cast<size_t>(k)];
        nd.face = scene.face(face[k]).id;
        nd.image = {image[3 * k], image[3 * k + 1], image[3 * k + 2]};
        nd.parent = parent[k];
        nd.depth = depth[k];
    }
    return out;
}

// ---------------------------------------------------------------------------
// Public single-pair predicates (src/vismatrix.cpp:160-225, 387-476)
// ---------------------------------------------------------------------------
bool mutually_front(const Face& a, const Face& b) {
    auto has_front_point = [](const Face& of, const Face& probe) {
        for (const Vec3& p : probe.poly.pts)
            if (signed_distance(of, p) > kEps) return true;
        return false;
    };
    return has_front_point(a, b) && has_front_point(b, a);
}

std::vector<PlaneTag> required_planes(const Face& ref, const Face& aim) {
    std::vector<PlaneTag> out;
    for (PlaneTag tag : {PlaneTag::XY, PlaneTag::YZ, PlaneTag::XZ}) {
        const auto sr = plane_segment(ref, tag);
        const auto sa = plane_segment(aim, tag);
        if (!sr || !sa) continue;
        const double d = std::abs(dot2(sr->normal, sa->normal));
        if (d >= 1.0 - 1e-9 || d <= 1e-9) out.push_back(tag);
    }
    return out;
}

namespace {
const char* plane_name(PlaneTag p) { return p == PlaneTag::XY ? "XY" : (p == PlaneTag::YZ ? "YZ" : "XZ"); }
}  // namespace

InterfaceRelation classify_relation_in_plane(const Face& ref, const Face& aim, PlaneTag plane) {
    const auto sr = plane_segment(ref, plane);
    const auto sa = plane_segment(aim, plane);
    if (!sr || !sa)
        throw VisibilityError("faces '" + ref.id + "' and '" + aim.id + "' do not both project to segments in plane " +
                              plane_name(plane));
    const double d = std::abs(dot2(sr->normal, sa->normal));
    InterfaceRelation rel;
    rel.plane = plane;
    rel.chain = {ref.id, aim.id};
    rel.chain_orientations = {ref.orientation, aim.orientation};
    if (d >= 1.0 - 1e-9) rel.kind = RelationKind::Parallel;
    else if (d <= 1e-9) rel.kind = RelationKind::Perpendicular;
    else
        throw VisibilityError("faces '" + ref.id + "' and '" + aim.id +
                              "' are neither parallel nor perpendicular in plane " + plane_name(plane));
    return rel;
}

InterfaceRelation classify_relation(const Face& ref, const Face& aim) {
    if (ref.id == aim.id) throw VisibilityError("reference and aim face must differ (got '" + ref.id + "')");
    if (ref.orientation == Orientation::Oblique || aim.orientation == Orientation::Oblique)
        throw VisibilityError("unsupported relation: face pair ('" + ref.id + "', '" + aim.id +
                              "') involves an oblique face");
    const auto planes = required_planes(ref, aim);
    if (planes.empty())
        throw VisibilityError("unsupported relation: faces '" + ref.id + "' and '" + aim.id +
                              "' share no working plane");
    return classify_relation_in_plane(ref, aim, planes.front());
}

SecondOrderResult second_order_check(const Face& original, const Face& mid, const Face& test,
                                     const InterVisMatrix& matrix, PlaneTag plane) {
    if (!matrix.find(1, original.id, mid.id, plane) || !matrix.find(1, mid.id, test.id, plane))
        throw VisibilityError("second-order check needs first-order entries for ('" + original.id + "','" + mid.id +
                              "') and ('" + mid.id + "','" + test.id + "') in plane " + plane_name(plane));
    const auto so = plane_segment(original, plane), sm = plane_segment(mid, plane), st = plane_segment(test, plane);
    if (!so || !sm || !st)
        throw VisibilityError(std::string("second-order check: missing segment projection in plane ") +
                              plane_name(plane));
    Segs segs;   // the three segments as a 3-face table
    segs.seg.assign(18 * 3, 0.0);
    segs.ok.assign(9, 0);
    const PlaneSegment* ps[3] = {&*so, &*sm, &*st};
    const int pl = static_cast<int>(plane);
    for (int f = 0; f < 3; ++f) {
        double* d = &segs.seg[(static_cast<size_t>(f) * 3 + pl) * 6];
        d[0] = ps[f]->a.x; d[1] = ps[f]->a.y; d[2] = ps[f]->b.x; d[3] = ps[f]->b.y;
        d[4] = ps[f]->normal.x; d[5] = ps[f]->normal.y;
        segs.ok[3 * f + pl] = 1;
    }
    ISet reach;
    SecondOrderResult r;
    r.verdict = second_order(segs, 0, 1, 2, plane, reach);
    if (r.verdict == ChainVerdict::Partial) r.reachable.assign(reach.begin(), reach.end());
    return r;
}

bool chain_triple_feasible(const Face& original, const Face& mid, const Face& test) {
    const Scene* sc = owner_of(mid);
    if (!sc || owner_of(original) != sc || owner_of(test) != sc)
        throw std::invalid_argument("chain_triple_feasible: faces must belong to one finalized rt::Scene");
    const int32_t t[3] = {original.index, mid.index, test.index};
    uint8_t ok = 0;
    check(visrt_triples_feasible(sc->device_scene(), 1, t, &ok, nullptr));
    return ok != 0;
}

std::vector<Path> accelerated_trace(const Scene& scene, const InterVisMatrix& matrix, const Vec3& tx, const Vec3& rx,
                                    int max_refl, bool allow_diffraction, TraceStats* stats) {
    const TraceAccelerator accel(scene, matrix, max_refl);
    return accel.trace(tx, rx, allow_diffraction, stats);
}

// ---------------------------------------------------------------------------
// EM consumer (src/em.cpp:194-235) over the GPU kernels
// ---------------------------------------------------------------------------
std::vector<RayGain> ray_gains(const Scene& scene, const std::vector<Path>& paths, const EmConfig& config) {
    if (config.frequency <= 0) throw EmError("frequency must be positive");
    const size_t n = scene.faces().size();
    std::vector<double> mat(2 * n);
    for (size_t f = 0; f < n; ++f) {
        const Material& m = scene.material(scene.face(static_cast<int>(f)).material);
        mat[2 * f] = m.permittivity;
        mat[2 * f + 1] = m.conductivity;
    }
    std::map<std::string, int> edge_index;
    std::vector<double> ab;
    std::vector<int32_t> ef;
    for (const Edge& e : scene.edges()) {
        edge_index.emplace(e.id, static_cast<int>(edge_index.size()));
        ab.insert(ab.end(), {e.a.x, e.a.y, e.a.z, e.b.x, e.b.y, e.b.z});
        ef.push_back(scene.face(e.faces[0]).index);
        ef.push_back(scene.face(e.faces[1]).index);
    }
    std::vector<visrt_path> vp(paths.size());
    for (size_t q = 0; q < paths.size(); ++q) {
        const Path& p = paths[q];
        visrt_path& o = vp[q];
        std::memset(&o, 0, sizeof(o));
        o.edge = -1;
        for (const Interaction& ia : p.interactions) {
            if (ia.kind == InteractionKind::Reflection) {
                if (o.nrefl >= 4) throw EmError("paths carry at most four reflections");
                o.faces[o.nrefl++] = scene.face(ia.id).index;
            } else {
                auto it = edge_index.find(ia.id);
                if (it == edge_index.end()) throw EmError("path references unknown edge '" + ia.id + "'");
                o.edge = it->second;
            }
        }
        for (size_t i = 0; i < p.points.size() && i < 7; ++i) {
            o.points[3 * i] = p.points[i].x;
            o.points[3 * i + 1] = p.points[i].y;
            o.points[3 * i + 2] = p.points[i].z;
        }
        o.length = p.length;
    }
    const visrt_em_config cfg{config.frequency, config.tx_gain_dbi, config.rx_gain_dbi,
                              config.polarization == Polarization::TM ? 1 : 0, 0};
    std::vector<double> amp(2 * paths.size() + 2), delay(paths.size() + 1);
    visrt_stats st{};
    const int rc = visrt_ray_gains(scene.device_scene(), static_cast<int64_t>(paths.size()), vp.data(), mat.data(),
                                   static_cast<int32_t>(ef.size() / 2), ab.empty() ? nullptr : ab.data(),
                                   ef.empty() ? nullptr : ef.data(), &cfg, amp.data(), delay.data(), &st, nullptr);
    if (rc == VISRT_E_VISIBILITY) throw EmError(visrt_last_error());
    check(rc);
    std::vector<RayGain> rays;
    for (size_t q = 0; q < paths.size(); ++q)
        rays.push_back({{amp[2 * q], amp[2 * q + 1]}, delay[q], paths[q].identity()});
    return rays;
}

ChannelStats channel_stats(const std::vector<RayGain>& rays) {   // src/em.cpp:209-235
    ChannelStats stats;
    stats.rays = rays;
    if (rays.empty()) {
        stats.outage = true;
        return stats;
    }
    double power = 0.0, m1 = 0.0, m2 = 0.0;
    for (const RayGain& r : rays) {
        const double p = std::norm(r.amplitude);
        power += p;
        m1 += p * r.delay;
        m2 += p * r.delay * r.delay;
    }
    if (power <= 0) {
        stats.outage = true;
        return stats;
    }
    stats.path_loss_db = -10.0 * std::log10(power);
    m1 /= power;
    m2 /= power;
    stats.rms_delay_spread = std::sqrt(std::max(0.0, m2 - m1 * m1));
    return stats;
}

}  // namespace rt
