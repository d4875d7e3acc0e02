// visrt-b200 C++ drop-in layer: the hot-path subset of the reference's public
// C++ API (namespace rt, /root/reference/proj/include/rt/*.hpp) re-created on
// top of the C-ABI (include/visrt.h). Same names, argument meaning and
// exception types/messages for:
//   Scene / Face / Building / plane_segment          include/rt/scene.hpp:38-106
//   occlusion_judgment, build_matrix, InterVisMatrix, mutually_front, required_planes,
//   classify_relation(_in_plane), second_order_check, chain_triple_feasible  include/rt/vismatrix.hpp:37-153
//   illuminated_region                                include/rt/vistable.hpp:116-117
//   TraceAccelerator / Path / TraceStats / image_tree include/rt/raytracer.hpp:25-118
//   point_vis_table, trajectory_vis_table, closest_diffraction_edge  include/rt/vistable.hpp:62-148
// Geometry is decided on the GPU (sm_100a kernels); the host materialises the
// string-keyed records (ids, angle records with atan2, aim images) exactly as
// the reference does. There is no CPU fallback for any hot-path decision.
#pragma once

#include <array>
#include <cmath>
#include <complex>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

struct visrt_scene;
struct visrt_tracer;

namespace rt {

inline constexpr double kEps = 1e-9;
inline constexpr double kSpeedOfLight = 299792458.0;

struct Vec3 {
    double x = 0.0, y = 0.0, z = 0.0;
    Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
    Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
    Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
};
struct Vec2 {
    double x = 0.0, y = 0.0;
};
enum class PlaneTag { XY, YZ, XZ };
enum class Orientation { Horizontal, Vertical, Oblique };

class SceneError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
class VisibilityError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
class PlacementError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

struct ConvexPolygon {
    std::vector<Vec3> pts;
    Vec3 normal;
    static ConvexPolygon from_points(std::vector<Vec3> pts);  // Newell normal
};

struct FaceLabels {
    std::string xy, vert;
};

struct Face {
    std::string id;
    std::string building;
    std::string material;
    ConvexPolygon poly;
    Orientation orientation = Orientation::Vertical;
    FaceLabels labels;
    int index = -1;
    const std::string& label(PlaneTag p) const {
        if (p == PlaneTag::XY) return labels.xy.empty() ? id : labels.xy;
        return labels.vert.empty() ? id : labels.vert;
    }
};

struct Edge {
    std::string id;
    Vec3 a, b;
    std::array<std::string, 2> faces;
    std::string building;
};

struct Building {
    std::string id;
    std::vector<Face> faces;
};

struct PlaneSegment {
    Vec2 a, b, normal;
};

/// include/rt/scene.hpp:21-25
struct Material {
    std::string name;
    double permittivity = 1.0;
    double conductivity = 0.0;
};

class Scene {
  public:
    std::vector<Material> materials;
    std::vector<Building> buildings;
    std::optional<Face> ground;
    const Material& material(const std::string& name) const;

    Scene() = default;
    Scene(const Scene&) = delete;             // faces() holds pointers into the scene
    Scene& operator=(const Scene&) = delete;
    Scene(Scene&& other);                     // re-indexes the moved faces (load_scene returns by value)
    ~Scene();

    /// Closed-shell scenes (reference semantics: indices, orientations, edges).
    void finalize();
    /// Facet soup (open boxes on tiled ground): no buildings, no edges.
    static std::unique_ptr<Scene> from_facets(const std::vector<std::string>& ids,
                                              const std::vector<std::vector<Vec3>>& rings);

    const std::vector<const Face*>& faces() const { return face_ptrs_; }
    const Face& face(int index) const { return *face_ptrs_.at(static_cast<size_t>(index)); }
    const Face& face(const std::string& id) const;
    const std::vector<Edge>& edges() const { return edges_; }
    bool inside_building(const Vec3& p) const;

    /// The device-resident copy (created on first use on CUDA device 0).
    visrt_scene* device_scene() const;

  private:
    std::vector<const Face*> face_ptrs_;
    std::vector<Face> soup_;
    std::map<std::string, int> face_index_;
    std::vector<Edge> edges_;
    mutable visrt_scene* dev_ = nullptr;
};

std::optional<PlaneSegment> plane_segment(const Face& face, PlaneTag plane);

/// The reference's JSON scene files (include/rt/scene.hpp:108-109,
/// src/scene.cpp:288-375): materials, shared vertex list, buildings of faces
/// (id, material, vertex indices, optional labels), optional ground face.
/// load_scene finalizes (same validation and SceneError messages);
/// save_scene interns vertices by exact coordinates in face order. A facet
/// soup (Scene::from_facets) has no JSON form: SceneError.
Scene load_scene(const std::string& path);
void save_scene(const Scene& scene, const std::string& path);

// ---------------------------------------------------------------------------
enum class RelationKind { Parallel, Perpendicular };
enum class ChainVerdict { Full, Partial, None };

struct InterfaceRelation {
    RelationKind kind = RelationKind::Parallel;
    PlaneTag plane = PlaneTag::XY;
    std::vector<std::string> chain;
    std::vector<Orientation> chain_orientations;
};
struct AngleRecord {
    std::string edge_id;
    Vec2 vertex, ref_dir, outward;
    double low = 0.0, high = 0.0;
};
struct AngularBouncingRange {
    AngleRecord at_a, at_b;
};
struct OcclusionVerdict {
    enum class Kind { Visible, PartiallyVisible, Occluded };
    Kind kind = Kind::Visible;
    std::vector<std::string> blockers;
};
struct InterVisEntry {
    int order = 1;
    std::string ref, aim;
    InterfaceRelation relation;
    AngularBouncingRange ranges;
    std::optional<AngularBouncingRange> criterion;
    ChainVerdict verdict = ChainVerdict::Full;
    std::vector<std::array<double, 2>> subranges;
    std::vector<std::string> blockers;
    std::vector<Vec3> aim_image;
};

class InterVisMatrix {
  public:
    int max_order() const { return max_order_; }
    const std::vector<InterVisEntry>& entries() const { return entries_; }
    std::vector<const InterVisEntry*> find(int order, const std::string& ref, const std::string& aim) const;
    const InterVisEntry* find(int order, const std::string& ref, const std::string& aim, PlaneTag plane) const;
    bool pair_admitted(const std::string& ref, const std::string& aim) const;
    std::vector<std::string> aims_of(const std::string& ref) const;
    void add(InterVisEntry entry);
    void set_max_order(int order) { max_order_ = order; }

  private:
    int max_order_ = 1;
    std::vector<InterVisEntry> entries_;
    std::map<std::tuple<int, std::string, std::string>, std::vector<size_t>> index_;
};

OcclusionVerdict occlusion_judgment(const Face& ref, const Face& aim, const Scene& scene);

/// Public predicates of include/rt/vismatrix.hpp:105-153 (single-pair helpers
/// of the matrix builder; the builder itself runs them batched on the GPU).
bool mutually_front(const Face& a, const Face& b);
std::vector<PlaneTag> required_planes(const Face& ref, const Face& aim);
InterfaceRelation classify_relation_in_plane(const Face& ref, const Face& aim, PlaneTag plane);
InterfaceRelation classify_relation(const Face& ref, const Face& aim);
struct SecondOrderResult {
    ChainVerdict verdict = ChainVerdict::None;
    std::vector<std::array<double, 2>> reachable;
};
SecondOrderResult second_order_check(const Face& original, const Face& mid, const Face& test,
                                     const InterVisMatrix& matrix, PlaneTag plane);
/// GPU (K7's exact predicate); the faces must belong to a finalized rt::Scene.
bool chain_triple_feasible(const Face& original, const Face& mid, const Face& test);
InterVisMatrix build_matrix(const Scene& scene, int max_order);
/// Binary matrix / pair-graph cache (replaces the text save_matrix /
/// load_matrix of include/rt/vismatrix.hpp:143-144): admitted pairs + order-2
/// chains; load re-derives every entry exactly as build_matrix does.
void save_matrix_cache(const InterVisMatrix& matrix, const Scene& scene, const std::string& path);
InterVisMatrix load_matrix_cache(const Scene& scene, const std::string& path);

// ---------------------------------------------------------------------------
struct PlaneIllumination {
    PlaneTag plane = PlaneTag::XY;
    Vec2 image, face_a, face_b, outward;
    double alpha_full = 0.0, beta_full = 0.0;
    std::array<double, 2> sub{0.0, 1.0};
    Vec2 sub_a, sub_b;
    double alpha = 0.0, beta = 0.0;
    bool clipped = false;
    std::vector<Vec2> clip_points;
};
struct IlluminatedRegion {
    std::string face;
    Vec3 source;
    std::vector<PlaneIllumination> planes;
    const PlaneIllumination* plane(PlaneTag tag) const {
        for (const auto& p : planes)
            if (p.plane == tag) return &p;
        return nullptr;
    }
};
std::optional<IlluminatedRegion> illuminated_region(const Vec3& source, const Face& face, const Scene& scene);
/// Batched form (one GPU call for every (source, face)): regions[k][f].
std::vector<std::vector<std::optional<IlluminatedRegion>>> illuminated_regions(const std::vector<Vec3>& sources,
                                                                               const Scene& scene);

/// include/rt/vistable.hpp:62-76
struct VisTableEntry {
    int order = 1;
    std::string parent, ref, aim;
    PlaneTag plane = PlaneTag::XY;
    std::string parent_display, ref_display, aim_display;
    ChainVerdict verdict = ChainVerdict::Full;
    std::vector<std::string> chain;
};
/// point_vis_table (include/rt/vistable.hpp:128-129): GPU regions + beam
/// cascade; matrix entries of order <= min(max_order, 2).
std::vector<VisTableEntry> point_vis_table(const Vec3& source, const InterVisMatrix& matrix, const Scene& scene,
                                           int max_order);

/// include/rt/scene.hpp:130-142 (the table-relevant part)
struct Trajectory {
    std::vector<Vec3> waypoints;
    std::vector<double> speeds;
    double total_length() const;
    Vec3 position_at(double s) const;
};
/// include/rt/vistable.hpp:82-93
struct MobileVisEntry {
    int order = 1;
    std::string node, node_display;
    double s_start = 0.0, s_end = 0.0;
    std::string label_start, label_end, parent, blockage;
};
inline constexpr double kTrajectoryStep = 0.5;
inline constexpr double kBoundaryTolerance = 1e-3;
/// trajectory_vis_table (include/rt/vistable.hpp:143-148): one GPU call.
std::vector<MobileVisEntry> trajectory_vis_table(const Trajectory& traj, const InterVisMatrix& matrix,
                                                 const Scene& scene, int max_order);
/// closest_diffraction_edge (include/rt/vistable.hpp:131-137)
std::optional<Edge> closest_diffraction_edge(const Vec3& receiver, const Scene& scene);
std::optional<Edge> closest_diffraction_edge(const Vec3& receiver, const Scene& scene, const InterVisMatrix& matrix);

// ---------------------------------------------------------------------------
/// include/rt/raytracer.hpp:51-61
struct ImageTreeNode {
    std::string face;
    Vec3 image;
    int parent = -1;
    int depth = 1;
};
std::vector<ImageTreeNode> image_tree(const Scene& scene, const Vec3& source, int max_depth);

enum class InteractionKind { Reflection, Diffraction };
struct Interaction {
    InteractionKind kind = InteractionKind::Reflection;
    std::string id;
    Vec3 point;
};
struct Path {
    std::vector<Interaction> interactions;
    Vec3 source, receiver;
    std::vector<Vec3> points;
    double length = 0.0, delay = 0.0;
    std::string identity() const;
};
struct TraceStats {
    long long nodes_expanded = 0, sequences_checked = 0, occlusion_tests = 0, paths_found = 0;
};

class TraceAccelerator {
  public:
    TraceAccelerator(const Scene& scene, const InterVisMatrix& matrix, int max_refl);
    ~TraceAccelerator();
    TraceAccelerator(const TraceAccelerator&) = delete;
    TraceAccelerator& operator=(const TraceAccelerator&) = delete;
    /// allow_diffraction: the receiver's closest diffraction edge adds the
    /// sequences ending at its Fermat point (facet soups have no edges).
    std::vector<Path> trace(const Vec3& tx, const Vec3& rx, bool allow_diffraction,
                            TraceStats* stats = nullptr) const;
    /// Batched form: one GPU expansion over every snapshot (rx.size() == 1: fixed receiver).
    std::vector<std::vector<Path>> trace_batch(const std::vector<Vec3>& tx, const std::vector<Vec3>& rx,
                                               std::vector<TraceStats>* stats = nullptr,
                                               bool allow_diffraction = false) const;
    int max_reflections() const { return max_refl_; }

  private:
    friend std::vector<Path> brute_force_trace(const Scene&, const Vec3&, const Vec3&, int, bool, TraceStats*);
    TraceAccelerator(const Scene& scene, int max_refl);   // brute force: no filter, no prune
    void set_edges(const Scene& scene);
    const Scene* scene_;
    int max_refl_;
    bool brute_ = false;
    visrt_tracer* tracer_ = nullptr;
};

/// accelerated_trace (include/rt/raytracer.hpp:121-124): one-shot TraceAccelerator.
std::vector<Path> accelerated_trace(const Scene& scene, const InterVisMatrix& matrix, const Vec3& tx,
                                    const Vec3& rx, int max_refl, bool allow_diffraction,
                                    TraceStats* stats = nullptr);

/// brute_force_trace (include/rt/raytracer.hpp:78-83): the unaccelerated image
/// method on the GPU tree (every face but the immediate repeat, no prune).
std::vector<Path> brute_force_trace(const Scene& scene, const Vec3& tx, const Vec3& rx, int max_refl,
                                    bool allow_diffraction, TraceStats* stats = nullptr);

// ---------------------------------------------------------------------------
/// EM consumer (include/rt/em.hpp:14-103), GPU kernels with CUDA's
/// transcendentals (tolerance-level agreement with the reference).
class EmError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
enum class Polarization { TE, TM };
struct EmConfig {
    double frequency = 5.5e9;
    double tx_gain_dbi = 0.0;
    double rx_gain_dbi = 0.0;
    Polarization polarization = Polarization::TE;
};
struct RayGain {
    std::complex<double> amplitude;
    double delay = 0.0;
    std::string path_id;
};
struct ChannelStats {
    bool outage = false;
    double path_loss_db = std::numeric_limits<double>::infinity();
    double rms_delay_spread = 0.0;
    std::vector<RayGain> rays;
};
std::vector<RayGain> ray_gains(const Scene& scene, const std::vector<Path>& paths, const EmConfig& config);
ChannelStats channel_stats(const std::vector<RayGain>& rays);

}  // namespace rt
