/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the visibility hot path.
 *
 * A plain-C restatement of the reference algorithm (arxiv 2501.02747 artifact,
 * /root/reference/proj), each function citing the reference file:line it
 * follows. Pinned against the compiled reference (oracle/_ref, see
 * oracle/Makefile) and the committed golden fixtures in tests/golden/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product path never does.
 */
#ifndef VISRT_ORACLE_H
#define VISRT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vo_scene vo_scene;

/* Facet soup in: rings of vertices, vert_off[n+1] prefix offsets. */
vo_scene* vo_scene_create(int32_t nfaces, const int32_t* vert_off, const double* verts);
void vo_scene_free(vo_scene* s);
int32_t vo_nfaces(const vo_scene* s);
/* Per-face ingest products: normal[3], orientation (0 H, 1 V, 2 O). */
int32_t vo_face_info(const vo_scene* s, int32_t i, double* normal, int32_t* orientation);
/* plane_segment: 1 + a.x a.y b.x b.y n.x n.y, or 0. */
int32_t vo_plane_segment(const vo_scene* s, int32_t i, int32_t plane, double* out6);

int32_t vo_segment_hits_face(const vo_scene* s, const double* a, const double* b, int32_t face);
int32_t vo_mutually_front(const vo_scene* s, int32_t i, int32_t j);
int32_t vo_required_planes(const vo_scene* s, int32_t i, int32_t j);   /* bitmask XY|YZ|XZ */
int32_t vo_prefilter(const vo_scene* s, int32_t i, int32_t j);         /* first_order_pair gate */
/* All i<j passing the gate, in (i, j) order, on `threads` pthreads. Two-call
 * sizing: out == NULL returns the count. */
int64_t vo_prefilter_all(const vo_scene* s, int32_t* out_i, int32_t* out_j, int64_t cap, int32_t threads);

/* occlusion_judgment: kind 0 Visible / 1 Partial / 2 Occluded. Blockers as a
 * sorted face-index list (the reference sorts ids as strings; callers map). */
int32_t vo_occlusion(const vo_scene* s, int32_t i, int32_t j, int32_t* blockers, int32_t cap,
                     int32_t* nblk);
/* Pair batch on `threads` pthreads: kind per pair (no blockers). */
int32_t vo_occlusion_batch(const vo_scene* s, int64_t npairs, const int32_t* pi, const int32_t* pj,
                           int8_t* kind, int32_t threads);
/* Sightline count S(i,j) as occlusion_judgment builds them. */
int32_t vo_sightline_count(const vo_scene* s, int32_t i, int32_t j);

/* illuminated_region subset: present (1), none (0), VisibilityError (-1);
 * per plane tag (3 slots by PlaneTag): has, sub[2], clipped. */
typedef struct {
    int32_t present;
    int32_t has[3];
    int32_t clipped[3];
    double sub[6];
} vo_region;
int32_t vo_illuminated_region(const vo_scene* s, const double* src, int32_t face, vo_region* out);

/* (3) TraceAccelerator::trace, allow_diffraction = false, for a soup scene
 * (no buildings, no edges, no oblique faces needed). Chain filter: order-1
 * continuations = admitted aims as CSR (off1[n+1], idx1 ascending per row),
 * order-2 continuations = CSR over the directed admitted pairs in the same
 * order (c2_off[npairs+1], c2_idx): the key (p, t) is the position of t in
 * p's aim list.
 * Paths: nrefl, faces[4], points[3*(nrefl+2)], length. Returns path count,
 * or -1 (PlacementError: tx ~ rx). stats: nodes, sequences, paths. */
typedef struct {
    int32_t nrefl;
    int32_t faces[4];
    double points[18];
    double length;
} vo_path;
int64_t vo_trace(const vo_scene* s, const int64_t* off1, const int32_t* idx1, const int64_t* c2_off,
                 const int32_t* c2_idx, int32_t max_refl, const double* tx, const double* rx, vo_path* out,
                 int64_t cap, int64_t* stats);

#ifdef __cplusplus
}
#endif
#endif
