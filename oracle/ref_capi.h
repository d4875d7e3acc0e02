/* TEST INFRASTRUCTURE ONLY — C-ABI of the compiled-reference adapter
 * (oracle/ref_capi.cpp -> oracle/_ref/libvisrt_ref.so). */
#ifndef VISRT_REF_CAPI_H
#define VISRT_REF_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t order;
    int32_t chain[5];
    int32_t chain_len;
    int32_t plane;
    int32_t kind;      /* 0 PAR, 1 PER */
    int32_t verdict;   /* 0 Full, 1 Partial */
    int32_t has_criterion;
    int32_t nblockers;
    int32_t nsub;
    int32_t naim_image;
    double ranges[12];     /* at_a: vertex.x, vertex.y, low, high, ref_dir.x, ref_dir.y; at_b: same */
    double criterion[4];   /* at_a low/high, at_b low/high */
    double sub[8];         /* up to 4 subranges */
    double aim_image[24];  /* up to 8 points */
    int32_t blockers[64];
    char edge_a[64];
    char edge_b[64];
} vref_entry;

typedef struct {
    int32_t present;      /* 0 none, 1 present, -1 VisibilityError */
    int32_t nplanes;
    int32_t plane[3];
    int32_t clipped[3];
    double sub[6];
    double image[6];
    double sub_ab[12];
    double angles[12];    /* alpha_full, beta_full, alpha, beta per plane */
} vref_region;

typedef struct {
    int32_t ninter;
    int32_t face[6];
    int32_t is_diff[6];
    double points[24];
    double length;
    double delay;
    char identity[256];
} vref_path;

typedef struct {
    int32_t order;
    int32_t chain[4];
    int32_t chain_len;
    int32_t aim;
    int32_t plane;
    int32_t verdict;
    char ref_display[32];
    char aim_display[32];
    char parent_display[32];
} vref_row;

typedef struct {
    int32_t order;
    int32_t pad;
    double s_start;
    double s_end;
    char node[64];
    char node_display[64];
    char label_start[16];
    char label_end[16];
    char parent[64];
    char blockage[64];
} vref_mobile_row;

const char* vref_last_error(void);
void* vref_scene_from_soup(int32_t nfaces, const int32_t* vert_off, const double* verts, const char* ids);
void* vref_scene_from_shells(int32_t nfaces, const int32_t* vert_off, const double* verts, const char* ids,
                             const int32_t* building, int32_t nbuildings, const char* building_ids);
void vref_scene_free(void* h);
int32_t vref_scene_save(void* h, const char* path);
int32_t vref_nfaces(void* h);
int32_t vref_nedges(void* h);
void* vref_scene_load(const char* path);
int32_t vref_face_export(void* h, int32_t idx, char* id, int32_t idcap, char* bld, int32_t bldcap, char* lab_xy,
                         char* lab_vert, int32_t labcap, double* pts, int32_t ptcap, double* normal);
int32_t vref_edge_export(void* h, int32_t idx, char* id, int32_t idcap, double* ab);
void* vref_build_matrix(void* h, int32_t order);
void vref_matrix_free(void* m);
void vref_matrix_set_max_order(void* m, int32_t order);
int64_t vref_matrix_size(void* m);
int32_t vref_matrix_entry(void* h, void* m, int64_t k, vref_entry* out);
int64_t vref_matrix_chains(void* h, void* m, int32_t order, int32_t* out, int64_t cap);
int32_t vref_occlusion(void* h, int32_t i, int32_t j, int32_t* blockers, int32_t cap, int32_t* nblk);
int32_t vref_illuminated_region(void* h, const double* src, int32_t face, vref_region* out);
int64_t vref_point_vis_table(void* h, void* m, const double* src, int32_t max_order, vref_row* rows, int64_t cap);
int64_t vref_trajectory_table(void* h, void* m, int32_t nwp, const double* wp, int32_t max_order,
                              vref_mobile_row* rows, int64_t cap);
int32_t vref_closest_edge(void* h, const double* rx);
int32_t vref_mutually_front(void* h, int32_t i, int32_t j);
int32_t vref_segments_blocked(void* h, int64_t n, const double* a, const double* b, uint8_t* blocked,
                              int32_t threads);
int32_t vref_required_planes(void* h, int32_t i, int32_t j);
int32_t vref_triple_feasible(void* h, int32_t p, int32_t t, int32_t a);
int32_t vref_chain_triple_feasible(void* h, int32_t p, int32_t t, int32_t a);
int64_t vref_trace_em(void* h, void* a, const double* tx, const double* rx, int32_t diffraction, double freq,
                      double tx_gain, double rx_gain, int32_t tm, double* amp, double* delay, double* stats3,
                      int64_t cap);
int64_t vref_image_tree(void* h, const double* src, int32_t depth, int32_t* face, int32_t* parent,
                        int32_t* dep, double* image, int64_t cap);
int64_t vref_brute_trace(void* h, const double* tx, const double* rx, int32_t max_refl, int32_t diffraction,
                         vref_path* out, int64_t cap, int64_t* stats);
void* vref_accel_create(void* h, void* m, int32_t max_refl);
void vref_accel_free(void* a);
int64_t vref_accel_trace(void* h, void* a, const double* tx, const double* rx, int32_t diffraction,
                         vref_path* out, int64_t cap, int64_t* stats);

#ifdef __cplusplus
}
#endif
#endif
