// Shared declarations of the (2) per-snapshot table kernels (regions.cu) for
// the other translation units that drive them (trajectory.cu).
#pragma once

#include <cuda_runtime.h>

#include "device.h"

namespace visrt {

// K4 task list. A launch decides `ntasks` (source k, face f) regions in one of
// three modes; region_task() below is the ONE mapping task t -> (k, f, list
// entry li, output slot) both region kernels use:
//   task_face == nullptr : all faces of every source, out[k * n + f]
//   paired == 0          : face list task_face[0..m) per source, out[k * m + li]
//   paired == 1          : query list, source t, face task_face[t], out[t]
// The walk order of the first two modes is `face_major`: 1 = consecutive tasks
// take one face (list entry) for consecutive sources (K4w's default: warps
// share blockers and cached lines), 0 = one source for consecutive faces.
struct RegionArgs {
    DevScene s;
    long long ntasks;
    const double* src;            // [nsrc][3]
    visrt_region* out;            // [ntasks]
    unsigned long long* counter;  // [0] cursor, [1] exact tests, [2] sightlines
    const int32_t* task_face = nullptr;
    int m = 0;
    int paired = 0;
    // presence only (K4w): present = every plane with a face_param has a
    // visible column (the scan stops at the first one; no refinement, no sub)
    // — exactly whether illuminated_region returns a region
    int presence_only = 0;
    const uint8_t* presence_of = nullptr;   // per face-list entry (list mode) / per task (paired)
    int chunk = 1;                          // K4w: consecutive tasks per warp grab (set by the launcher)
    int face_major = 1;                     // walk order of the all-faces / face-list modes (see above)
    int fan = 1;                            // K4w: refine run boundaries with fan candidate lists
    float4* cone_buf = nullptr;             // K4w: per-warp cone lists (cone_cap entries of 2 float4), set by the launcher
    int cone_cap = 0;
    unsigned long long* refine_count = nullptr;   // K4w: [0] RefineTasks appended at the buffer front, [1] refine
                                                  // kernel cursor, [2] heavy ones at its end (launcher, zeroed)
    void* refine_tasks = nullptr;                 // K4w: RefineTask[ntasks] (regions.cu), set by the launcher
};

struct RegionTask {
    long long k, li, out;   // source, face-list entry (list mode, else 0), output slot
    int f;                  // face
};

__device__ __forceinline__ RegionTask region_task(const RegionArgs& a, long long t, int n) {
    RegionTask r;
    r.li = 0;
    if (a.paired) {
        r.k = t;
        r.f = a.task_face[t];
        r.out = t;
        return r;
    }
    const long long per = a.task_face ? a.m : n;   // faces per source
    if (a.face_major) {
        const long long nsrc = a.ntasks / per;
        r.li = t / nsrc;
        r.k = t - r.li * nsrc;
    } else {
        r.k = t / per;
        r.li = t - r.k * per;
    }
    r.f = a.task_face ? a.task_face[r.li] : static_cast<int>(r.li);
    r.out = r.k * per + r.li;
    if (!a.task_face) r.li = 0;
    return r;
}

// K5 (TableBuilder::reach for order 1/2 chains). Dense: every (source k,
// entry e), region of face f at regions[k * rstride + slot[f]] (slot NULL:
// slot[f] = f, rstride = n), output bit e of row k. Paired: query t = (source
// t, entry t, region t), output bit t of row 0.
struct BeamArgs {
    DevScene s;
    long long nsrc, nent;
    const double* src;
    const visrt_region* regions;
    const visrt_entry* ent;
    uint32_t* row_bits;            // [nsrc][words]
    uint32_t* full_bits;
    int32_t words;
    const int32_t* slot = nullptr;
    int rstride = 0;
    int paired = 0;
};

struct Cov {
    int verdict;                   // 0 Full, 1 Partial, 2 None
    double lo, hi;
};

// beam_coverage, src/vistable.cpp:225-272 (apex, window [wa, wb], outward; target qa->qb)
__device__ inline Cov beam_coverage(double apx, double apy, double wax, double way, double wbx, double wby,
                                    double ox, double oy, double qax, double qay, double qbx, double qby) {
    Cov r{2, 0.0, 0.0};
    const double eax = dsub(wax, apx), eay = dsub(way, apy);
    const double ebx = dsub(wbx, apx), eby = dsub(wby, apy);
    const double inner = dsub(dmul(eax, eby), dmul(eay, ebx));
    const double scale = dmul(__dsqrt_rn(dadd(dmul(eax, eax), dmul(eay, eay))),
                              __dsqrt_rn(dadd(dmul(ebx, ebx), dmul(eby, eby))));
    const double smax1 = scale < 1.0 ? 1.0 : scale;   // std::max(scale, 1.0)
    if (fabs(inner) <= dmul(1e-14, smax1)) return r;
    const double sgn = inner > 0.0 ? 1.0 : -1.0;
    double lo = 0.0, hi = 1.0;
    auto apply = [&](double c0, double c1) {
        if (fabs(c1) <= dmul(1e-15, dadd(fabs(c0), 1.0))) {
            if (c0 < 0.0) {
                lo = 1.0;
                hi = 0.0;
            }
            return;
        }
        const double t = __ddiv_rn(-c0, c1);
        if (c1 > 0.0) lo = (lo < t) ? t : lo;     // std::max(lo, t)
        else hi = (t < hi) ? t : hi;              // std::min(hi, t)
    };
    const double dqx = dsub(qbx, qax), dqy = dsub(qby, qay);
    apply(dadd(dmul(dsub(qax, wax), ox), dmul(dsub(qay, way), oy)), dadd(dmul(dqx, ox), dmul(dqy, oy)));
    const double rax = dsub(qax, apx), ray = dsub(qay, apy);
    apply(dmul(sgn, dsub(dmul(eax, ray), dmul(eay, rax))), dmul(sgn, dsub(dmul(eax, dqy), dmul(eay, dqx))));
    apply(dmul(-sgn, dsub(dmul(ebx, ray), dmul(eby, rax))), dmul(-sgn, dsub(dmul(ebx, dqy), dmul(eby, dqx))));
    if (dsub(hi, lo) <= 1e-12) return r;
    r.lo = lo;
    r.hi = hi;
    if (lo <= 1e-9 && hi >= 1.0 - 1e-9) {
        r.verdict = 0;
        r.lo = 0.0;
        r.hi = 1.0;
    } else {
        r.verdict = 1;
    }
    return r;
}

__device__ __forceinline__ void proj(int pl, double x, double y, double z, double& u, double& v) {
    if (pl == 0) { u = x; v = y; }
    else if (pl == 1) { u = y; v = z; }
    else { u = x; v = z; }
}

cudaError_t launch_point_regions(const RegionArgs& a, int device, cudaStream_t st);
cudaError_t launch_beam_rows(const BeamArgs& a, cudaStream_t st);
// counter[0] must be zero (work cursor); counter[1] += exact tests
cudaError_t launch_segments_clear(const DevScene& s, long long nseg, const double* A, const double* B,
                                  uint8_t* clear, unsigned long long* counter, int device, cudaStream_t st);

// closest_diffraction_edge for a batch of receivers (imagetree.cu): out_edge[r]
// = edge index or -1; ms / tests of the GPU sightline sweep.
void closest_edges(const visrt_scene* sc, int64_t nrx, const double* rx_xyz, int32_t nedges, const double* edge_ab,
                   const int32_t* edge_rank, int32_t* out_edge, float* ms, int64_t* tests, cudaStream_t st);

}  // namespace visrt
