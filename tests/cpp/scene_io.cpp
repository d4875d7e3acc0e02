// rt::load_scene / rt::save_scene (the drop-in layer, paper_2501_02747_b200/cpp)
// against the UNMODIFIED reference's (visrt_ref::, oracle/ref_capi.h) on the
// reference's own scene files: every face (id, building, labels, vertex ring,
// Newell normal — doubles compared with ==), every edge (id, endpoints), the
// saved JSON text, and the SceneError messages of unreadable / invalid files.
// Usage: scene_io <scene.json> <tmpdir>. Exit code = number of mismatches.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "../../oracle/ref_capi.h"
#include "../../paper_2501_02747_b200/cpp/rt.hpp"

static int g_bad = 0;
#define EXPECT(cond, what)                                                  \
    do {                                                                    \
        if (!(cond)) {                                                      \
            if (g_bad < 20) std::cerr << "MISMATCH " << what << std::endl;  \
            ++g_bad;                                                        \
        }                                                                   \
    } while (0)

static std::string slurp(const std::string& p) {
    std::ifstream in(p);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

static void compare(const rt::Scene& s, void* ref, const std::string& tag) {
    const int n = vref_nfaces(ref);
    EXPECT(static_cast<int>(s.faces().size()) == n, tag << " face count");
    for (int i = 0; i < n && i < static_cast<int>(s.faces().size()); ++i) {
        char id[128], bld[128], lx[128], lv[128];
        double pts[3 * 64], nrm[3];
        const int nv = vref_face_export(ref, i, id, 128, bld, 128, lx, lv, 128, pts, 64, nrm);
        const rt::Face& f = s.face(i);
        EXPECT(f.id == id && f.building == bld && f.labels.xy == lx && f.labels.vert == lv, tag << " face " << i);
        EXPECT(static_cast<int>(f.poly.pts.size()) == nv, tag << " ring size " << f.id);
        for (int k = 0; k < nv && k < static_cast<int>(f.poly.pts.size()); ++k)
            EXPECT(f.poly.pts[k].x == pts[3 * k] && f.poly.pts[k].y == pts[3 * k + 1] &&
                       f.poly.pts[k].z == pts[3 * k + 2], tag << " vertex " << f.id << "#" << k);
        EXPECT(f.poly.normal.x == nrm[0] && f.poly.normal.y == nrm[1] && f.poly.normal.z == nrm[2],
               tag << " normal " << f.id);
        EXPECT(f.index == i, tag << " index " << f.id);
    }
    const int ne = vref_nedges(ref);
    EXPECT(static_cast<int>(s.edges().size()) == ne, tag << " edge count");
    for (int e = 0; e < ne && e < static_cast<int>(s.edges().size()); ++e) {
        char id[128];
        double ab[6];
        vref_edge_export(ref, e, id, 128, ab);
        const rt::Edge& g = s.edges()[e];
        EXPECT(g.id == id && g.a.x == ab[0] && g.a.y == ab[1] && g.a.z == ab[2] && g.b.x == ab[3] &&
                   g.b.y == ab[4] && g.b.z == ab[5], tag << " edge " << e);
    }
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::string path = argv[1], tmp = argv[2];
    void* ref = vref_scene_load(path.c_str());
    if (!ref) {
        std::cerr << "reference load failed: " << vref_last_error() << std::endl;
        return 3;
    }
    rt::Scene s = rt::load_scene(path);
    compare(s, ref, "load");
    // save: both layers write the same JSON text
    rt::save_scene(s, tmp + "/ours.json");
    vref_scene_save(ref, (tmp + "/ref.json").c_str());
    EXPECT(slurp(tmp + "/ours.json") == slurp(tmp + "/ref.json"), "saved JSON text differs");
    // round trip through our own file
    rt::Scene s2 = rt::load_scene(tmp + "/ours.json");
    compare(s2, ref, "reload");
    // error messages (SceneError) of a missing and of an invalid file
    auto msg_of = [](auto fn) -> std::string {
        try {
            fn();
        } catch (const rt::SceneError& e) {
            return e.what();
        } catch (const std::exception& e) {
            return std::string("other: ") + e.what();
        }
        return "no throw";
    };
    const std::string missing = tmp + "/does_not_exist.json";
    std::string ours = msg_of([&] { rt::load_scene(missing); });
    void* r2 = vref_scene_load(missing.c_str());
    EXPECT(!r2 && ours == vref_last_error(), "missing-file message: " << ours);
    {
        std::ofstream bad(tmp + "/bad.json");
        bad << "{\"materials\": [{\"name\": \"m\", \"permittivity\": 0.5, \"conductivity\": 0}]}";
    }
    ours = msg_of([&] { rt::load_scene(tmp + "/bad.json"); });
    r2 = vref_scene_load((tmp + "/bad.json").c_str());
    EXPECT(!r2 && ours == vref_last_error(), "invalid-material message: " << ours << " vs " << vref_last_error());
    vref_scene_free(ref);
    std::cout << "OK " << g_bad << " mismatches, " << s.faces().size() << " faces, " << s.edges().size() << " edges"
              << std::endl;
    return g_bad;
}
