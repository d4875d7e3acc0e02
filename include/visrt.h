/* visrt-b200 — C-ABI of the B200-native visibility pre-processing hot path.
 *
 * The reference (arxiv 2501.02747 artifact, /root/reference/proj) has no FFI;
 * its boundary is the C++ API of namespace rt. Each entry point below is what
 * that API's hot-path functions bind to (see INTEGRATION.md for the C++ drop-in
 * layer and the ctypes binding):
 *
 *   visrt_scene_create        <- Scene::finalize / facet ingest
 *                                (include/rt/scene.hpp:81-88, src/scene.cpp:65-182,
 *                                 src/geom.cpp:126-140, src/scene.cpp:213-254)
 *   visrt_pair_visibility     <- build_matrix pair loop + occlusion_judgment
 *                                (include/rt/vismatrix.hpp:113,141;
 *                                 src/vismatrix.cpp:253-302, 597-675)
 *   visrt_pair_detail         <- occlusion_judgment verdict kind + blocker set
 *                                (src/vismatrix.cpp:275-301)
 *   visrt_point_regions       <- illuminated_region for (snapshot, face) batches
 *                                (include/rt/vistable.hpp:116-117, src/vistable.cpp:287-334)
 *   visrt_point_tables        <- point_vis_table (include/rt/vistable.hpp:128-129)
 *   visrt_chain_reach         <- TableBuilder::reach / MobileSampler::member (src/vistable.cpp:404-467)
 *   visrt_trajectory_table    <- trajectory_vis_table (include/rt/vistable.hpp:143-148)
 *   visrt_closest_edges       <- closest_diffraction_edge (include/rt/vistable.hpp:131-137)
 *   visrt_chain_triples       <- build_matrix chain growth (src/vismatrix.cpp:715-797)
 *   visrt_tracer_* / visrt_trace <- TraceAccelerator::trace, brute_force_trace / Engine::expand +
 *                                resolve_sequence (include/rt/raytracer.hpp:78-118, src/raytracer.cpp:174-493)
 *   visrt_image_tree          <- image_tree (include/rt/raytracer.hpp:51-61)
 *
 * Conventions: plain pointers and sizes; caller-owned output buffers; every
 * call returns a status (0 ok) and never throws; the message of the last
 * failure on the calling thread is visrt_last_error(). Status codes map to
 * the reference exception types: 1 VisibilityError, 2 PlacementError,
 * 3 SceneError, 4 CUDA error, 5 capacity/usage error.
 * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 */
#ifndef VISRT_H
#define VISRT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VISRT_OK 0
#define VISRT_E_VISIBILITY 1
#define VISRT_E_PLACEMENT 2
#define VISRT_E_SCENE 3
#define VISRT_E_CUDA 4
#define VISRT_E_USAGE 5

#define VISRT_MAX_VERTS 8

typedef struct visrt_scene visrt_scene;

/* Facet soup (or closed-shell scene) in host memory. */
typedef struct {
    int32_t nfaces;
    const int32_t* vert_off;   /* [nfaces+1] prefix offsets, in vertices            */
    const double* verts;       /* [3*vert_off[nfaces]] xyz per vertex, rings in order */
    const int32_t* building;   /* [nfaces] building index, -1 = none; NULL = soup   */
} visrt_facets_v1;

typedef struct {
    int64_t pairs;             /* unordered pairs evaluated                          */
    int64_t candidates;        /* pairs passing the first_order_pair prefilter       */
    int64_t admitted;          /* pairs not Occluded (bit set)                       */
    double  tests_alg;         /* sum S(i,j)*(N-2) over evaluated pairs (reference work) */
    int64_t tests_exec;        /* segment-vs-facet tests the kernel executed         */
    float   ms;                /* device time of the call (CUDA events)              */
    int64_t sweeps;            /* culled occluder sweeps started (one per sightline)  */
    int64_t tiles;             /* 64-occluder tiles culled by lanes (SAT work / 64)   */
} visrt_stats;

const char* visrt_last_error(void);
int visrt_version(void);

/* Ingest on the host with the reference's arithmetic, upload the facet SoA to
 * device `device`. */
int visrt_scene_create(const visrt_facets_v1* facets, int device, visrt_scene** out);
void visrt_scene_destroy(visrt_scene* scene);
int visrt_scene_nfaces(const visrt_scene* scene);
/* Host copies of ingest products: normal[3n], orientation[n] (0 H, 1 V, 2 O),
 * plane segments seg[n*3*6] (a.x a.y b.x b.y n.x n.y), seg_ok[n*3]. Any NULL skipped. */
int visrt_scene_ingest(const visrt_scene* scene, double* normal, int32_t* orientation,
                       double* seg, int32_t* seg_ok);
/* Bytes the scene upload copied host->device (the e2e H2D accounting). */
int64_t visrt_scene_upload_bytes(const visrt_scene* scene);
/* Measured device FP64 / FP32 arithmetic peaks (non-FMA DADD+DMUL ops/s and
 * FFMA-counted flop/s) from a short microbenchmark on `device`. */
int visrt_measure_peaks(int device, double* fp64_ops_per_s, double* fp32_flops_per_s);

/* (1) Inter-visibility matrix.
 * flags: VISRT_PAIRS_ALL        — (B) every i<j, bit = occlusion verdict != Occluded;
 *        VISRT_PAIRS_PREFILTERED — (A) candidates of first_order_pair's gate only
 *                                 (non-oblique, mutually_front, required_planes != {}).
 * bits: row-major N x ceil(N/64) uint64 words, symmetric (bit (i,j) and (j,i)).
 * Device-resident variant writes into scene-owned memory: visrt_matrix_bits_device(). */
#define VISRT_PAIRS_ALL 0x1u
#define VISRT_PAIRS_PREFILTERED 0x2u
int visrt_pair_visibility(visrt_scene* scene, uint32_t flags, uint64_t* bits_host,
                          visrt_stats* stats, void* stream);
/* Row block of the (B) matrix: only the pairs (i, j), i < j, with row0 <= i < row1 are
 * decided (the build_matrix pair loop's outer range, src/vismatrix.cpp:640-675, cut into
 * blocks). bits is still the full N x ceil(N/64) matrix, zero outside the block's pairs and
 * symmetric inside, so the blocks of a partition OR (or integer-add: disjoint bits) together
 * into the full matrix — the strong-scaling shard of one scene over several GPUs
 * (dist.pair_row_blocks gives blocks of equal pair count). flags must be VISRT_PAIRS_ALL;
 * stats count the block's pairs and reference tests. */
int visrt_pair_visibility_rows(visrt_scene* scene, uint32_t flags, int32_t row0, int32_t row1,
                               uint64_t* bits_host, visrt_stats* stats, void* stream);
const uint64_t* visrt_matrix_bits_device(const visrt_scene* scene);
/* Candidate list of the last PREFILTERED call (ordered by (i, j)), with the
 * verdict bit per candidate. Two-call sizing: pass NULL to get the count. */
int64_t visrt_candidates(const visrt_scene* scene, int32_t* ci, int32_t* cj, uint8_t* admitted);

/* Verdict kind (0 Visible, 1 PartiallyVisible, 2 Occluded) and blocker sets for
 * a pair list (ref = ci, aim = cj). blockers: CSR (blk_off[npairs+1], blk_idx)
 * sorted by face index; pass blk_idx = NULL to size (blk_off still filled). */
int visrt_pair_detail(visrt_scene* scene, int64_t npairs, const int32_t* ci, const int32_t* cj,
                      int8_t* kind, int64_t* blk_off, int32_t* blk_idx, int64_t blk_cap,
                      visrt_stats* stats, void* stream);

/* (2) Per-snapshot point regions: illuminated_region(source, face) for every
 * (source k, face f). Per (k, f): present (1 / 0 none / -1 source on plane),
 * per plane tag t in {XY, YZ, XZ}: has[t], clipped[t], sub[2t], sub[2t+1]. */
typedef struct {
    int8_t present;
    int8_t has[3];
    int8_t clipped[3];
    int8_t pad;
    double sub[6];
} visrt_region;
int visrt_point_regions(visrt_scene* scene, int64_t nsrc, const double* src_xyz,
                        visrt_region* out, visrt_stats* stats, void* stream);

/* (2) Per-snapshot point tables (point_vis_table rows, src/vistable.cpp:478-521)
 * for a list of matrix entries of order 1..4: entry e = (order, chain[0..2],
 * plane) with chain = reflectors..., aim. For every (source k, entry e) the
 * kernels decide whether TableBuilder::reach(reflectors) succeeds (the row
 * exists) and whether the beam is Full in the entry's plane, from the GPU
 * regions (illuminated_region) and the exact beam cascade (beam_coverage,
 * src/vistable.cpp:225-272, 432-467). Output bitsets row_bits/full_bits:
 * [nsrc][ceil(nent/32)] uint32 (bit e of source k). regions_out (optional):
 * the regions as visrt_point_regions would return them. */
typedef struct {
    int32_t order;        /* 1..4 */
    int32_t chain[5];     /* reflectors chain[0..order-1], aim chain[order] */
    int32_t plane;        /* the entry's working plane (PlaneTag) */
} visrt_entry;
int visrt_point_tables(visrt_scene* scene, int64_t nsrc, const double* src_xyz, int64_t nent,
                       const visrt_entry* entries, uint32_t* row_bits, uint32_t* full_bits,
                       visrt_region* regions_out, visrt_stats* stats, void* stream);

/* Batched sightline_clear (src/vistable.cpp:38-44 with skip = -1, i.e.
 * Occluder::clear semantics): clear[k] = no face blocks the open segment
 * a[k] -> b[k]. */
int visrt_segments_clear(visrt_scene* scene, int64_t nseg, const double* a_xyz, const double* b_xyz,
                         uint8_t* clear, visrt_stats* stats, void* stream);

/* chain_triple_feasible(original, mid, test) (include/rt/vismatrix.hpp:131,
 * src/vismatrix.cpp:457-476) for an explicit list of face triples. */
int visrt_triples_feasible(visrt_scene* scene, int64_t n, const int32_t* triples, uint8_t* feasible, void* stream);

/* TableBuilder::reach for a query list (src/vistable.cpp:404-430, 432-467):
 * query q = (source src_xyz[q], reflector chain chains[q].chain[0..order-1],
 * order 1..4; chain[order] and plane name an entry whose plane decides
 * full[q]). reach[q] = the beam reaches the last reflector (the row /
 * MobileSampler::member test); full[q] (may be NULL) = Full in that plane. */
int visrt_chain_reach(visrt_scene* scene, int64_t nq, const double* src_xyz, const visrt_entry* chains,
                      uint8_t* reach, uint8_t* full, visrt_stats* stats, void* stream);

/* (2) Trajectory visibility table: trajectory_vis_table(traj, matrix, scene,
 * max_order) (include/rt/vistable.hpp:143-148, src/vistable.cpp:822-960) with
 * MobileSampler (681-812). Inputs: the route waypoints, the matrix entries
 * (order <= max_order used; max_order 1..4) in matrix order, and the string
 * orders the reference sorts by, as integer ranks (any order-consistent
 * integers; equal strings must get equal ranks):
 *   key_rank[9n+1]   : face id of f at [f], corner node "<id>#k" at [n + 8f + k],
 *                      "transmitter" at [9n]        (SigKey order, row node order)
 *   parent_rank[n+1] : label(XY) of f at [f], "transmitter" at [n]   (row parent order)
 *   building_rank[n] : building_of(f) ("ground" for faces without building)
 * Rows come back in the reference's order; labels are integers: boundary i is
 * "P<i>" (+ "'" when prime_*), 0 is "-". blockage is a building rank or -1 ("-").
 * stats: pairs = samples, candidates = boundaries, admitted = rows,
 * tests_exec = exact predicate tests, sweeps = kernel launches, ms = device time. */
typedef struct {
    const int32_t* key_rank;
    const int32_t* parent_rank;
    const int32_t* building_rank;
} visrt_names;
typedef struct {
    int32_t order;
    int32_t node;          /* face index */
    int32_t vertex;        /* corner k of a "<id>#k" node, -1 = face node */
    int32_t parent;        /* face index, -1 = "transmitter" */
    double s_start, s_end;
    int32_t label_start, label_end;
    int32_t prime_start, prime_end;
    int32_t blockage;
    int32_t pad;
} visrt_mobile_row;
typedef struct visrt_mobile_table visrt_mobile_table;
int visrt_trajectory_table(visrt_scene* scene, int32_t nwp, const double* waypoints, int64_t nent,
                           const visrt_entry* entries, int32_t max_order, const visrt_names* names,
                           visrt_mobile_table** out, visrt_stats* stats, void* stream);
/* Copy up to cap rows (rows may be NULL); returns the row count. */
int64_t visrt_mobile_table_rows(const visrt_mobile_table* table, visrt_mobile_row* rows, int64_t cap);
void visrt_mobile_table_destroy(visrt_mobile_table* table);

/* Binary matrix / pair-graph cache (replaces the text
 * format of save_matrix / load_matrix, src/vismatrix.cpp:805-968): the
 * admitted order-1 bits + the feasible order-2 triples, tied to the scene by a
 * fingerprint (load on another scene -> status 3 SceneError). Host-only
 * handles (device < 0) are accepted. load: bits and triples NULL = header
 * only (max_order, ntriples); else cap must hold the cached triples. */
int visrt_cache_save(const char* path, const visrt_scene* scene, int32_t max_order, const uint64_t* admitted_bits,
                     int64_t ntriples, const int32_t* triples);
int visrt_cache_load(const char* path, const visrt_scene* scene, int32_t* max_order, uint64_t* admitted_bits,
                     int32_t* triples, int64_t cap, int64_t* ntriples);

/* Order-2 chains of build_matrix(scene, 2) (src/vismatrix.cpp:715-797): every
 * triple p->t->a of admitted pairs that passes chain_triple_feasible and
 * second_order_check in each shared working plane. admitted_bits NULL = the
 * scene's device bits of the last PREFILTERED call. out == NULL: count only.
 * Triples are returned sorted by (p, t, a). */
int visrt_chain_triples(visrt_scene* scene, const uint64_t* admitted_bits, int32_t* out, int64_t cap,
                        int64_t* ntriples, visrt_stats* stats, void* stream);

/* (3) Image-tree expansion (TraceAccelerator::trace, allow_diffraction = false).
 * The chain filter (build_chain_filter, src/raytracer.cpp:319-340) is given as
 * the admitted order-1 bit matrix (pair_admitted; NULL = the scene's device
 * bits of the last PREFILTERED visrt_pair_visibility) plus the order-2 chains
 * (triples p->t->a, required for max_refl 3). Per snapshot k (tx[k], rx[k] or
 * rx[0] when rx_fixed) the accelerated image tree is expanded level by level
 * on the GPU; results stay in the tracer until fetched. */
typedef struct visrt_tracer visrt_tracer;
int visrt_tracer_create(visrt_scene* scene, int max_refl, const uint64_t* admitted_bits,
                        int64_t ntriples, const int32_t* triples, visrt_tracer** out);
void visrt_tracer_destroy(visrt_tracer* tracer);
typedef struct {
    int32_t nrefl;         /* 0..4 */
    int32_t faces[4];      /* reflecting faces, source side first            */
    int32_t edge;          /* diffraction edge index (last interaction), -1 none */
    int32_t snap;
    int32_t pad;
    double points[21];     /* tx, reflection points..., [diffraction point], rx */
    double length;
} visrt_path;
typedef struct {
    int64_t nodes;         /* image-tree nodes expanded (TraceStats::nodes_expanded) */
    int64_t sequences;     /* sequences resolved (TraceStats::sequences_checked)     */
    int64_t paths;         /* paths found (TraceStats::paths_found)                  */
    int64_t leg_tests;     /* exact segment-vs-face tests run on path legs            */
    float   ms;            /* device time of the whole batch                          */
} visrt_trace_stats;
/* flags: VISRT_TRACE_RX_FIXED — one receiver rx[0] for every snapshot;
 * VISRT_TRACE_DIFFRACTION — allow_diffraction = true: per snapshot the
 * closest diffraction edge of the receiver (closest_diffraction_edge over the
 * edges of visrt_tracer_set_edges) adds Engine::attempt's second sequence
 * per node, ending at the edge's Fermat point (src/raytracer.cpp:174-192,
 * 367, 383-394). */
#define VISRT_TRACE_RX_FIXED 0x1
#define VISRT_TRACE_DIFFRACTION 0x2
/* VISRT_TRACE_BRUTE_FORCE — brute_force_trace (src/raytracer.cpp:488-493): the
 * unaccelerated image method, every face but the immediate repeat at every
 * level, no chain filter and no image prune (Engine with filter = nullptr). */
#define VISRT_TRACE_BRUTE_FORCE 0x4
int visrt_trace(visrt_tracer* tracer, int64_t nsnap, const double* tx, const double* rx,
                int flags, visrt_trace_stats* stats, void* stream);
/* One fixed interaction sequence (SequenceKey, src/raytracer.cpp:528-552):
 * reflecting faces (source side first) + optional final diffraction edge. */
typedef struct {
    int32_t nrefl;         /* 0..4 */
    int32_t faces[4];
    int32_t edge;          /* -1: the path ends at the receiver */
} visrt_seqkey;
/* resolve_keys (src/raytracer.cpp:554-570), the dynamic-run re-solve: for
 * every sample k (tx[k], rx[k] or rx[0] with VISRT_TRACE_RX_FIXED) and every
 * key q in key_off[k]..key_off[k+1]-1, resolve_sequence(keys[q]) at the new
 * endpoints: ok[q] = a valid path exists (unfolding + every leg clear), and
 * paths[q] (may be NULL) = that path (snap = k). edge_ab: the scene's edges. */
int visrt_resolve_keys(visrt_scene* scene, int64_t nsamp, const double* tx, const double* rx, int flags,
                       const int64_t* key_off, const visrt_seqkey* keys, int32_t nedges, const double* edge_ab,
                       uint8_t* ok, visrt_path* paths, visrt_stats* stats, void* stream);

/* EM consumer of the path sets: ray_gains and
 * channel_stats (include/rt/em.hpp:92-103, src/em.cpp:194-235). Per path
 * (visrt_path as returned by the tracer): complex amplitude amp[2q..2q+1]
 * (re, im; relative to unit transmit power and the antenna gains) and delay.
 * face_material: [nfaces][2] relative permittivity, conductivity (S/m);
 * edges as for the tracer plus their two adjacent faces (edge_faces[2e], the
 * 0-face first). Transcendentals are CUDA's: parity is tolerance-based.
 * Errors (the reference's EmError) map to status 1. */
typedef struct {
    double frequency;      /* Hz */
    double tx_gain_dbi;
    double rx_gain_dbi;
    int32_t polarization;  /* 0 TE, 1 TM */
    int32_t pad;
} visrt_em_config;
int visrt_ray_gains(visrt_scene* scene, int64_t npaths, const visrt_path* paths, const double* face_material,
                    int32_t nedges, const double* edge_ab, const int32_t* edge_faces, const visrt_em_config* config,
                    double* amp, double* delay, visrt_stats* stats, void* stream);
/* channel_stats per snapshot over its rays path_off[k]..path_off[k+1]: outage,
 * path loss -10 log10(sum |a|^2) (inf on outage) and the power-weighted RMS
 * delay spread. */
int visrt_channel_stats(visrt_scene* scene, int64_t nsnap, const int64_t* path_off, const double* amp,
                        const double* delay, int8_t* outage, double* path_loss_db, double* rms_delay_spread,
                        void* stream);

/* The scene's edges for diffraction (Scene::edges, include/rt/scene.hpp:85-95):
 * edge e = (a, b) at edge_ab[6e..6e+5]; edge_rank[e] = order of its id string. */
int visrt_tracer_set_edges(visrt_tracer* tracer, int32_t nedges, const double* edge_ab, const int32_t* edge_rank);
/* Unfiltered mirror hierarchy image_tree(scene, source, max_depth)
 * (include/rt/raytracer.hpp:51-61, src/raytracer.cpp:458-486): nodes in the
 * reference's depth-first order — face index, parent node (-1 at depth 1),
 * depth, image[3]. Two-call sizing: all outputs NULL returns the count in
 * *nnodes; otherwise cap must be >= the count. */
int visrt_image_tree(visrt_scene* scene, const double* src, int32_t max_depth, int32_t* face, int32_t* parent,
                     int32_t* depth, double* image, int64_t cap, int64_t* nnodes, visrt_stats* stats,
                     void* stream);

/* closest_diffraction_edge(receiver, scene) (include/rt/vistable.hpp:131-137,
 * src/vistable.cpp:529-561) for nrx receivers over the scene's edges (edge e:
 * a = edge_ab[6e..6e+2], b = edge_ab[6e+3..6e+5], in the scene's edge order;
 * edge_rank[e] = order of its id string, for the tie-break). out_edge[r] =
 * edge index, -1 = none visible. */
int visrt_closest_edges(visrt_scene* scene, int64_t nrx, const double* rx_xyz, int32_t nedges,
                        const double* edge_ab, const int32_t* edge_rank, int32_t* out_edge, visrt_stats* stats,
                        void* stream);

/* Fetch the last visrt_trace results: per-snapshot CSR (path_off[nsnap+1]),
 * paths grouped by snapshot, each group sorted by face sequence; nodes[nsnap]
 * per-snapshot node counts. Any pointer may be NULL; returns the path count. */
int64_t visrt_trace_results(const visrt_tracer* tracer, int64_t* path_off, visrt_path* paths,
                            int64_t path_cap, int64_t* nodes);
/* Per snapshot of the last visrt_trace: the closest diffraction edge used
 * (-1: none / diffraction off). Returns the snapshot count. */
int64_t visrt_trace_snapshot_edges(const visrt_tracer* tracer, int32_t* snap_edge);

#ifdef __cplusplus
}
#endif
#endif
