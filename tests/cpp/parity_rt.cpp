// Drop-in parity: the visrt-b200 C++ layer (namespace rt, GPU underneath)
// against the UNMODIFIED reference (visrt_ref::, through oracle/ref_capi.h) on
// one scene file written by tests/test_cpp_dropin.py. Every compared field is
// bit-exact (doubles compared with ==). Exit code = number of mismatches.
//
// Scene file:  nfaces nbuildings / building ids / per face: id b nv x y z ... /
//              nsrc / sources / ntrace / tx ty tz rx ry rz / max_order
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "../../oracle/ref_capi.h"
#include "../../paper_2501_02747_b200/cpp/rt.hpp"

static int g_bad = 0;
#define EXPECT(cond, what)                                                     \
    do {                                                                       \
        if (!(cond)) {                                                         \
            if (g_bad < 20) std::cerr << "MISMATCH " << what << std::endl;     \
            ++g_bad;                                                           \
        }                                                                      \
    } while (0)

// hex-float token (libstdc++ streams do not parse hexfloat input)
static double rd(std::istream& in) {
    std::string tok;
    in >> tok;
    return std::strtod(tok.c_str(), nullptr);
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ifstream in(argv[1]);
    int n = 0, nb = 0;
    in >> n >> nb;
    std::vector<std::string> bids(nb), ids(n);
    std::vector<int> bidx(n);
    std::vector<std::vector<rt::Vec3>> rings(n);
    for (auto& b : bids) in >> b;
    std::vector<int32_t> off{0};
    std::vector<double> verts;
    for (int i = 0; i < n; ++i) {
        int nv = 0;
        in >> ids[i] >> bidx[i] >> nv;
        for (int k = 0; k < nv; ++k) {
            rt::Vec3 p;
            p.x = rd(in);
            p.y = rd(in);
            p.z = rd(in);
            rings[i].push_back(p);
            verts.insert(verts.end(), {p.x, p.y, p.z});
        }
        off.push_back(off.back() + nv);
    }
    int nsrc = 0;
    in >> nsrc;
    std::vector<rt::Vec3> src(nsrc);
    for (auto& s : src) {
        s.x = rd(in);
        s.y = rd(in);
        s.z = rd(in);
    }
    int ntr = 0;
    in >> ntr;
    std::vector<std::pair<rt::Vec3, rt::Vec3>> tr(ntr);
    for (auto& t : tr) {
        t.first.x = rd(in);
        t.first.y = rd(in);
        t.first.z = rd(in);
        t.second.x = rd(in);
        t.second.y = rd(in);
        t.second.z = rd(in);
    }
    int max_order = 2;
    in >> max_order;

    // --- both scenes -----------------------------------------------------
    std::string idcat, bcat;
    for (auto& s : ids) idcat += s + '\0';
    for (auto& s : bids) bcat += s + '\0';
    std::unique_ptr<rt::Scene> owned;
    rt::Scene* mine = nullptr;
    void* ref = nullptr;
    if (nb > 0) {
        owned = std::make_unique<rt::Scene>();
        owned->materials.push_back({"concrete", 5.31, 0.139});   // as vref_scene_from_shells
        owned->buildings.resize(nb);
        for (int b = 0; b < nb; ++b) owned->buildings[b].id = bids[b];
        for (int i = 0; i < n; ++i) {
            rt::Face f;
            f.id = ids[i];
            f.material = "concrete";
            f.poly = rt::ConvexPolygon::from_points(rings[i]);
            if (bidx[i] >= 0) owned->buildings[bidx[i]].faces.push_back(std::move(f));
            else owned->ground = std::move(f);
        }
        owned->finalize();
        ref = vref_scene_from_shells(n, off.data(), verts.data(), idcat.c_str(), bidx.data(), nb, bcat.c_str());
    } else {
        owned = rt::Scene::from_facets(ids, rings);
        ref = vref_scene_from_soup(n, off.data(), verts.data(), idcat.c_str());
    }
    mine = owned.get();
    if (!ref) {
        std::cerr << "reference scene: " << vref_last_error() << std::endl;
        return 99;
    }
    EXPECT(static_cast<int>(mine->faces().size()) == vref_nfaces(ref), "face count");
    auto id_of = [&](int i) { return mine->face(i).id; };

    // --- build_matrix ----------------------------------------------------
    const rt::InterVisMatrix M = rt::build_matrix(*mine, max_order);
    void* RM = vref_build_matrix(ref, max_order);
    const int64_t ne = vref_matrix_size(RM);
    EXPECT(static_cast<int64_t>(M.entries().size()) == ne, "entry count " << M.entries().size() << " vs " << ne);
    for (int64_t k = 0; k < ne && k < static_cast<int64_t>(M.entries().size()); ++k) {
        vref_entry r;
        vref_matrix_entry(ref, RM, k, &r);
        const rt::InterVisEntry& e = M.entries()[static_cast<size_t>(k)];
        std::ostringstream w;
        w << "entry " << k;
        EXPECT(e.order == r.order, w.str() << " order");
        EXPECT(static_cast<int>(e.relation.chain.size()) == r.chain_len, w.str() << " chain len");
        for (int c = 0; c < r.chain_len && c < static_cast<int>(e.relation.chain.size()); ++c)
            EXPECT(e.relation.chain[c] == id_of(r.chain[c]), w.str() << " chain");
        EXPECT(static_cast<int>(e.relation.plane) == r.plane, w.str() << " plane");
        EXPECT(static_cast<int>(e.relation.kind) == r.kind, w.str() << " kind");
        EXPECT(static_cast<int>(e.verdict) == r.verdict, w.str() << " verdict");
        const rt::AngleRecord* recs[2] = {&e.ranges.at_a, &e.ranges.at_b};
        for (int q = 0; q < 2; ++q) {
            const double* d = r.ranges + 6 * q;
            EXPECT(recs[q]->vertex.x == d[0] && recs[q]->vertex.y == d[1], w.str() << " vertex");
            EXPECT(recs[q]->low == d[2] && recs[q]->high == d[3], w.str() << " angles");
            EXPECT(recs[q]->ref_dir.x == d[4] && recs[q]->ref_dir.y == d[5], w.str() << " ref_dir");
        }
        EXPECT(e.ranges.at_a.edge_id == r.edge_a && e.ranges.at_b.edge_id == r.edge_b, w.str() << " edge ids");
        EXPECT(e.criterion.has_value() == (r.has_criterion != 0), w.str() << " criterion presence");
        if (e.criterion && r.has_criterion)
            EXPECT(e.criterion->at_a.low == r.criterion[0] && e.criterion->at_a.high == r.criterion[1] &&
                       e.criterion->at_b.low == r.criterion[2] && e.criterion->at_b.high == r.criterion[3],
                   w.str() << " criterion");
        EXPECT(static_cast<int>(e.subranges.size()) == r.nsub, w.str() << " subranges");
        for (int q = 0; q < r.nsub && q < static_cast<int>(e.subranges.size()); ++q)
            EXPECT(e.subranges[q][0] == r.sub[2 * q] && e.subranges[q][1] == r.sub[2 * q + 1], w.str() << " sub");
        EXPECT(static_cast<int>(e.blockers.size()) == r.nblockers, w.str() << " blocker count");
        for (int q = 0; q < r.nblockers && q < static_cast<int>(e.blockers.size()); ++q)
            EXPECT(e.blockers[q] == id_of(r.blockers[q]), w.str() << " blocker");
        EXPECT(static_cast<int>(e.aim_image.size()) == r.naim_image, w.str() << " aim image size");
        for (int q = 0; q < r.naim_image && q < static_cast<int>(e.aim_image.size()); ++q)
            EXPECT(e.aim_image[q].x == r.aim_image[3 * q] && e.aim_image[q].y == r.aim_image[3 * q + 1] &&
                       e.aim_image[q].z == r.aim_image[3 * q + 2],
                   w.str() << " aim image");
    }
    std::cout << "build_matrix(" << max_order << "): " << ne << " entries compared" << std::endl;

    // --- binary matrix cache round trip: every entry re-derived identically ---
    {
        const std::string cpath = std::string(argv[1]) + ".cache";
        rt::save_matrix_cache(M, *mine, cpath);
        const rt::InterVisMatrix MC = rt::load_matrix_cache(*mine, cpath);
        EXPECT(MC.max_order() == M.max_order() && MC.entries().size() == M.entries().size(), "cache entry count");
        for (size_t k = 0; k < M.entries().size() && k < MC.entries().size(); ++k) {
            const rt::InterVisEntry& x = M.entries()[k];
            const rt::InterVisEntry& y = MC.entries()[k];
            EXPECT(x.order == y.order && x.relation.chain == y.relation.chain && x.relation.plane == y.relation.plane &&
                       x.relation.kind == y.relation.kind && x.verdict == y.verdict && x.blockers == y.blockers &&
                       x.subranges == y.subranges && x.ranges.at_a.low == y.ranges.at_a.low &&
                       x.ranges.at_b.high == y.ranges.at_b.high && x.aim_image.size() == y.aim_image.size() &&
                       x.criterion.has_value() == y.criterion.has_value(),
                   "cache entry " << k);
        }
        std::cout << "matrix cache: " << MC.entries().size() << " entries re-derived" << std::endl;
    }

    // --- public single-pair predicates ----------------------------------------
    {
        int npp = 0;
        for (int i = 0; i < n; i += 3)
            for (int j = 0; j < n; j += 7) {
                if (i == j) continue;
                const rt::Face& a = mine->face(i);
                const rt::Face& b = mine->face(j);
                EXPECT(rt::mutually_front(a, b) == (vref_mutually_front(ref, i, j) != 0), "mutually_front " << i << "," << j);
                int m = 0;
                for (rt::PlaneTag t : rt::required_planes(a, b)) m |= 1 << static_cast<int>(t);
                EXPECT(m == vref_required_planes(ref, i, j), "required_planes " << i << "," << j);
                const int c = (i + 2 * j + 1) % n;
                if (c != i && c != j)
                    EXPECT(rt::chain_triple_feasible(a, b, mine->face(c)) ==
                               (vref_chain_triple_feasible(ref, i, j, c) != 0),
                           "chain_triple_feasible " << i << "," << j << "," << c);
                ++npp;
            }
        std::cout << "mutually_front / required_planes / chain_triple_feasible: " << npp << " cases compared" << std::endl;
    }

    // --- occlusion_judgment (every 5th pair) -------------------------------
    int npj = 0;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; j += 5) {
            const rt::OcclusionVerdict v = rt::occlusion_judgment(mine->face(i), mine->face(j), *mine);
            int32_t blk[4096];
            int32_t nblk = 0;
            const int k = vref_occlusion(ref, i, j, blk, 4096, &nblk);
            EXPECT(static_cast<int>(v.kind) == k, "verdict " << i << "," << j);
            EXPECT(static_cast<int>(v.blockers.size()) == nblk, "blockers " << i << "," << j);
            for (int q = 0; q < nblk && q < static_cast<int>(v.blockers.size()); ++q)
                EXPECT(v.blockers[q] == id_of(blk[q]), "blocker id " << i << "," << j);
            ++npj;
        }
    std::cout << "occlusion_judgment: " << npj << " pairs compared" << std::endl;

    // --- illuminated_region (every field, angles included) ---------------
    const auto regs = rt::illuminated_regions(src, *mine);
    for (int s = 0; s < nsrc; ++s)
        for (int f = 0; f < n; ++f) {
            vref_region r;
            const double sp[3] = {src[s].x, src[s].y, src[s].z};
            vref_illuminated_region(ref, sp, f, &r);
            const auto& g = regs[s][f];
            EXPECT(g.has_value() == (r.present == 1), "region presence " << s << "," << f);
            if (!g || r.present != 1) continue;
            EXPECT(static_cast<int>(g->planes.size()) == r.nplanes, "region planes " << s << "," << f);
            for (int p = 0; p < r.nplanes && p < static_cast<int>(g->planes.size()); ++p) {
                const rt::PlaneIllumination& pi = g->planes[p];
                EXPECT(static_cast<int>(pi.plane) == r.plane[p], "plane tag");
                EXPECT(pi.sub[0] == r.sub[2 * p] && pi.sub[1] == r.sub[2 * p + 1], "sub " << s << "," << f);
                EXPECT(pi.clipped == (r.clipped[p] != 0), "clipped");
                EXPECT(pi.image.x == r.image[2 * p] && pi.image.y == r.image[2 * p + 1], "image");
                EXPECT(pi.sub_a.x == r.sub_ab[4 * p] && pi.sub_a.y == r.sub_ab[4 * p + 1] &&
                           pi.sub_b.x == r.sub_ab[4 * p + 2] && pi.sub_b.y == r.sub_ab[4 * p + 3],
                       "sub_a/sub_b");
                EXPECT(pi.alpha_full == r.angles[4 * p] && pi.beta_full == r.angles[4 * p + 1] &&
                           pi.alpha == r.angles[4 * p + 2] && pi.beta == r.angles[4 * p + 3],
                       "boundary angles " << s << "," << f);
            }
        }
    std::cout << "illuminated_region: " << nsrc << " sources x " << n << " faces compared" << std::endl;

    // --- point_vis_table, image_tree, closest_diffraction_edge per source ---
    const int tab_order = max_order < 2 ? max_order : 2;
    std::vector<vref_row> rrows(1 << 16);
    for (int s = 0; s < nsrc; ++s) {
        const double sp[3] = {src[s].x, src[s].y, src[s].z};
        const auto rows = rt::point_vis_table(src[s], M, *mine, tab_order);
        const int64_t nrr = vref_point_vis_table(ref, RM, sp, tab_order, rrows.data(), 1 << 16);
        EXPECT(static_cast<int64_t>(rows.size()) == nrr, "point_vis_table rows " << s);
        for (int64_t q = 0; q < nrr && q < static_cast<int64_t>(rows.size()); ++q) {
            const rt::VisTableEntry& g = rows[static_cast<size_t>(q)];
            const vref_row& r = rrows[static_cast<size_t>(q)];
            EXPECT(g.order == r.order && static_cast<int>(g.chain.size()) == r.chain_len, "table row " << q);
            for (int c = 0; c < r.chain_len && c < static_cast<int>(g.chain.size()); ++c)
                EXPECT(g.chain[c] == id_of(r.chain[c]), "table chain");
            EXPECT(g.aim == id_of(r.aim) && static_cast<int>(g.plane) == r.plane, "table aim/plane");
            EXPECT(static_cast<int>(g.verdict) == r.verdict, "table verdict " << s << "," << q);
            EXPECT(g.ref_display == r.ref_display && g.aim_display == r.aim_display &&
                       g.parent_display == r.parent_display,
                   "table displays " << g.ref_display << "/" << r.ref_display);
        }
        const auto tree = rt::image_tree(*mine, src[s], 2);
        std::vector<int32_t> tf(1 << 20), tp(1 << 20), td(1 << 20);
        std::vector<double> ti(3 << 20);
        const int64_t nt = vref_image_tree(ref, sp, 2, tf.data(), tp.data(), td.data(), ti.data(), 1 << 20);
        EXPECT(static_cast<int64_t>(tree.size()) == nt, "image_tree size " << s);
        for (int64_t q = 0; q < nt && q < static_cast<int64_t>(tree.size()); ++q) {
            const rt::ImageTreeNode& g = tree[static_cast<size_t>(q)];
            EXPECT(g.face == id_of(tf[q]) && g.parent == tp[q] && g.depth == td[q], "image_tree node");
            EXPECT(g.image.x == ti[3 * q] && g.image.y == ti[3 * q + 1] && g.image.z == ti[3 * q + 2], "image");
        }
        const auto edge = rt::closest_diffraction_edge(src[s], *mine);
        const int32_t re = vref_closest_edge(ref, sp);
        EXPECT(edge.has_value() == (re >= 0), "closest edge presence " << s);
        if (edge && re >= 0) EXPECT(edge->id == mine->edges()[static_cast<size_t>(re)].id, "closest edge id");
    }
    std::cout << "point_vis_table / image_tree / closest_diffraction_edge: " << nsrc << " sources compared"
              << std::endl;

    // --- trajectory_vis_table along each trace's tx -> rx -----------------
    std::vector<vref_mobile_row> mrows(1 << 14);
    for (int t = 0; t < ntr; ++t) {
        rt::Trajectory traj;
        traj.waypoints = {tr[t].first, tr[t].second};
        traj.speeds = {1.0};
        if (traj.total_length() <= rt::kEps) continue;
        const auto rows = rt::trajectory_vis_table(traj, M, *mine, tab_order);
        const double wp[6] = {tr[t].first.x, tr[t].first.y, tr[t].first.z,
                              tr[t].second.x, tr[t].second.y, tr[t].second.z};
        const int64_t nm = vref_trajectory_table(ref, RM, 2, wp, tab_order, mrows.data(), 1 << 14);
        EXPECT(static_cast<int64_t>(rows.size()) == nm, "trajectory rows " << t << ": " << rows.size() << " vs " << nm);
        for (int64_t q = 0; q < nm && q < static_cast<int64_t>(rows.size()); ++q) {
            const rt::MobileVisEntry& g = rows[static_cast<size_t>(q)];
            const vref_mobile_row& r = mrows[static_cast<size_t>(q)];
            EXPECT(g.order == r.order && g.node == r.node && g.node_display == r.node_display, "mobile node " << q);
            EXPECT(g.s_start == r.s_start && g.s_end == r.s_end, "mobile s " << q);
            EXPECT(g.label_start == r.label_start && g.label_end == r.label_end, "mobile labels " << q);
            EXPECT(g.parent == r.parent && g.blockage == r.blockage, "mobile parent/blockage " << q);
        }
    }
    std::cout << "trajectory_vis_table: " << ntr << " routes compared" << std::endl;

    // --- TraceAccelerator up to max_order (+1 via set_max_order) ----------
    rt::InterVisMatrix M2 = M;
    M2.set_max_order(max_order + 1 <= 3 ? max_order + 1 : max_order);
    vref_matrix_set_max_order(RM, M2.max_order());
    for (int order = 1; order <= M2.max_order(); ++order) {
        rt::TraceAccelerator acc(*mine, M2, order);
        void* RA = vref_accel_create(ref, RM, order);
        for (int t = 0; t < 2 * ntr; ++t) {
            const bool diff = t >= ntr;   // second pass: allow_diffraction = true
            if (diff && mine->edges().empty()) break;
            const auto& trc = tr[t % ntr];
            rt::TraceStats st;
            const auto paths = acc.trace(trc.first, trc.second, diff, &st);
            std::vector<vref_path> rp(16384);
            int64_t rst[4];
            const double tx[3] = {trc.first.x, trc.first.y, trc.first.z};
            const double rx[3] = {trc.second.x, trc.second.y, trc.second.z};
            const int64_t np = vref_accel_trace(ref, RA, tx, rx, diff ? 1 : 0, rp.data(), 16384, rst);
            EXPECT(static_cast<int64_t>(paths.size()) == np, "path count order " << order << " trace " << t);
            if (order <= 2 && static_cast<int64_t>(paths.size()) == np && np > 0) {
                // EM consumer: GPU ray_gains vs the reference's, relative 1e-9
                rt::EmConfig cfg;
                cfg.frequency = 5.5e9;
                cfg.polarization = (t % 2) ? rt::Polarization::TM : rt::Polarization::TE;
                const auto rays = rt::ray_gains(*mine, paths, cfg);
                std::vector<double> ramp(2 * np), rdl(np), rst3(3);
                vref_trace_em(ref, RA, tx, rx, diff ? 1 : 0, cfg.frequency, 0.0, 0.0, (t % 2) ? 1 : 0, ramp.data(),
                              rdl.data(), rst3.data(), np);
                for (int64_t q = 0; q < np; ++q) {
                    const std::complex<double> rr(ramp[2 * q], ramp[2 * q + 1]);
                    EXPECT(std::abs(rays[static_cast<size_t>(q)].amplitude - rr) <= 1e-9 * std::abs(rr),
                           "ray gain " << q << " " << rays[static_cast<size_t>(q)].path_id);
                    EXPECT(rays[static_cast<size_t>(q)].delay == rdl[static_cast<size_t>(q)], "ray delay");
                }
                const rt::ChannelStats cs = rt::channel_stats(rays);
                EXPECT(cs.outage == (rst3[0] != 0.0), "channel outage");
                if (!cs.outage) EXPECT(std::abs(cs.path_loss_db - rst3[1]) <= 1e-9 * std::abs(rst3[1]), "path loss");
            }
            EXPECT(st.nodes_expanded == rst[0] && st.sequences_checked == rst[1], "trace stats " << order << "," << t);
            for (int64_t q = 0; q < np && q < static_cast<int64_t>(paths.size()); ++q) {
                const rt::Path& p = paths[static_cast<size_t>(q)];
                EXPECT(p.identity() == rp[q].identity, "identity " << p.identity() << " vs " << rp[q].identity);
                EXPECT(p.length == rp[q].length && p.delay == rp[q].delay, "length/delay");
                for (size_t v = 0; v < p.points.size(); ++v)
                    EXPECT(p.points[v].x == rp[q].points[3 * v] && p.points[v].y == rp[q].points[3 * v + 1] &&
                               p.points[v].z == rp[q].points[3 * v + 2],
                           "path point");
            }
        }
        vref_accel_free(RA);
        // brute_force_trace on the first traces (the unpruned tree grows as N^order)
        for (int t = 0; t < ntr && t < 2 && (order <= 2 || n <= 200); ++t) {
            rt::TraceStats st;
            const auto paths = rt::brute_force_trace(*mine, tr[t].first, tr[t].second, order, false, &st);
            std::vector<vref_path> rp(16384);
            int64_t rst[4];
            const double tx[3] = {tr[t].first.x, tr[t].first.y, tr[t].first.z};
            const double rx[3] = {tr[t].second.x, tr[t].second.y, tr[t].second.z};
            const int64_t np = vref_brute_trace(ref, tx, rx, order, 0, rp.data(), 16384, rst);
            EXPECT(static_cast<int64_t>(paths.size()) == np, "brute path count " << order << "," << t);
            EXPECT(st.nodes_expanded == rst[0] && st.sequences_checked == rst[1], "brute stats " << order << "," << t);
            for (int64_t q = 0; q < np && q < static_cast<int64_t>(paths.size()); ++q)
                EXPECT(paths[static_cast<size_t>(q)].identity() == rp[q].identity &&
                           paths[static_cast<size_t>(q)].length == rp[q].length,
                       "brute path " << order << "," << t);
        }
    }
    std::cout << "TraceAccelerator: orders 1.." << M2.max_order() << " x " << ntr
              << " traces compared (+ allow_diffraction where the scene has edges)" << std::endl;
    vref_matrix_free(RM);
    vref_scene_free(ref);
    std::cout << (g_bad ? "FAIL " : "OK ") << g_bad << " mismatches" << std::endl;
    return g_bad > 255 ? 255 : g_bad;
}
