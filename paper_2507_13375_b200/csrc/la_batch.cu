// GPU conflict-free net batching.
//
// Reading R31 of the paper's batching (§III-A l.224-226, Alg. 1 l.257-259):
// nets are assigned in parallel within a batch; this build forms batches that
// are CONFLICT-FREE, which makes the batched result identical to sequential
// assignment in priority order:
//   footprint(j) = unit 2D edges of net j's route U GCells of its LA-tree nodes
//   batch(j)     = 1 + max batch over earlier-priority nets sharing a footprint
//                  element, 0 if none  (longest path in the predecessor DAG).
// K1: radix-sort (element << 32 | rank) keys (CUB DeviceRadixSort, a library
//     sort primitive).  K2: successor edges between consecutive keys of the same
//     element, CSR by source, then Kahn frontiers: a net enters round r exactly
//     when its last predecessor left round r-1, i.e. r = its longest-path depth.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "la_internal.h"

namespace gapla {
namespace {

__global__ void k_edges_count(const uint64_t *__restrict__ keys, int64_t n, int32_t *__restrict__ outdeg,
                              int32_t *__restrict__ indeg) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i + 1 >= n) return;
    uint64_t a = keys[i], b = keys[i + 1];
    if ((a >> 32) != (b >> 32)) return;
    atomicAdd(outdeg + (uint32_t)a, 1);
    atomicAdd(indeg + (uint32_t)b, 1);
}

__global__ void k_edges_fill(const uint64_t *__restrict__ keys, int64_t n, const int64_t *__restrict__ off,
                             int32_t *__restrict__ cursor, int32_t *__restrict__ succ) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i + 1 >= n) return;
    uint64_t a = keys[i], b = keys[i + 1];
    if ((a >> 32) != (b >> 32)) return;
    uint32_t u = (uint32_t)a;
    int32_t slot = atomicAdd(cursor + u, 1);
    succ[off[u] + slot] = (int32_t)(uint32_t)b;
}

__global__ void k_frontier0(const int32_t *__restrict__ indeg, int64_t n, int32_t *__restrict__ batch,
                            int32_t *__restrict__ front, int32_t *__restrict__ count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (indeg[i] == 0) {
        batch[i] = 0;
        front[atomicAdd(count, 1)] = (int32_t)i;
    }
}

__global__ void k_frontier_step(const int32_t *__restrict__ front, int32_t nfront, const int64_t *__restrict__ off,
                                const int32_t *__restrict__ succ, int32_t *__restrict__ indeg,
                                int32_t *__restrict__ batch, int32_t round, int32_t *__restrict__ next,
                                int32_t *__restrict__ count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nfront) return;
    int32_t u = front[i];
    for (int64_t e = off[u]; e < off[u + 1]; ++e) {
        int32_t v = succ[e];
        if (atomicSub(indeg + v, 1) == 1) {
            batch[v] = round + 1;
            next[atomicAdd(count, 1)] = v;
        }
    }
}

__global__ void k_widen(const int32_t *__restrict__ a, int64_t *__restrict__ b, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}

// Forest-order DAG: position p holds the net of rank r = rank_of_pos[p].
__global__ void k_dag_deg(const int64_t *__restrict__ off_r, const int32_t *__restrict__ indeg_r,
                          const int64_t *__restrict__ rank_of_pos, int64_t n, int64_t *__restrict__ deg_p,
                          int32_t *__restrict__ indeg_p) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t r = rank_of_pos[p];
    deg_p[p] = off_r[r + 1] - off_r[r];
    indeg_p[p] = indeg_r[r];
}

__global__ void k_dag_fill(const int64_t *__restrict__ off_r, const int32_t *__restrict__ succ_r,
                           const int64_t *__restrict__ rank_of_pos, const int32_t *__restrict__ pos_of_rank,
                           const int64_t *__restrict__ off_p, int64_t n, int32_t *__restrict__ succ_p) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t r = rank_of_pos[p];
    int64_t o = off_p[p];
    for (int64_t e = off_r[r]; e < off_r[r + 1]; ++e) succ_p[o++] = pos_of_rank[succ_r[e]];
}

__global__ void k_inverse(const int64_t *__restrict__ rank_of_pos, int64_t n, int32_t *__restrict__ pos_of_rank) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < n) pos_of_rank[rank_of_pos[p]] = (int32_t)p;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() { if (p) dfree(p); }
    template <class T> T *as() { return static_cast<T *>(p); }
    cudaError_t alloc(size_t bytes) { return dmalloc(&p, bytes ? bytes : 16); }
};

#define BCK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

}  // namespace

void DagDev::release() {
    if (off) dfree(off);
    if (succ) dfree(succ);
    if (indeg) dfree(indeg);
    off = nullptr; succ = nullptr; indeg = nullptr;
    n = n_edges = 0;
}

// Footprint keys (element << 32 | rank) of every input net's as-built footprint elements, in place.
__global__ void k_fp_keys(const uint64_t *__restrict__ fp, const int64_t *__restrict__ start,
                          const int32_t *__restrict__ rank, int64_t n, uint64_t *keys) {
    const int64_t net = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (net >= n) return;
    const uint64_t r = (uint32_t)rank[net];
    for (int64_t j = start[net]; j < start[net + 1]; ++j) keys[j] = (fp[j] << 32) | r;
}

cudaError_t launch_fp_keys(const uint64_t *fp, const int64_t *start, const int32_t *rank, int64_t n, uint64_t *keys,
                           cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_fp_keys<<<nblk(n, 256), 256, 0, s>>>(fp, start, rank, n, keys);
    return cudaGetLastError();
}

cudaError_t gpu_conflict_batches(const uint64_t *h_keys, const uint64_t *d_keys, int64_t n_keys, int elem_bits,
                                 int64_t n_nets, std::vector<int32_t> &batch_of_rank, int32_t &n_batches,
                                 cudaStream_t s, int64_t *launches, DagDev *dag) {
    batch_of_rank.assign(n_nets, 0);
    n_batches = n_nets > 0 ? 1 : 0;
    if (n_nets == 0) return cudaSuccess;
    DevBuf kin, kout, tmp, outdeg, indeg, off, cursor, succ, batch, fa, fb, cnt;
    BCK(kin.alloc(8 * n_keys));
    BCK(kout.alloc(8 * n_keys));
    if (d_keys) BCK(cudaMemcpyAsync(kin.p, d_keys, 8 * n_keys, cudaMemcpyDeviceToDevice, s));
    else BCK(pinned_copy(kin.p, h_keys, 8 * n_keys, cudaMemcpyHostToDevice));   // pinned pipeline (the allocation synced)
    // K1: sort (element, rank) pairs
    size_t tmp_bytes = 0;
    int end_bit = 32 + elem_bits;
    BCK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, kin.as<uint64_t>(), kout.as<uint64_t>(), n_keys, 0,
                                       end_bit, s));
    size_t scan_bytes = 0;
    BCK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int64_t *)nullptr, (int64_t *)nullptr, n_nets + 1, s));
    BCK(tmp.alloc(std::max(tmp_bytes, scan_bytes)));
    BCK(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, kin.as<uint64_t>(), kout.as<uint64_t>(), n_keys, 0, end_bit,
                                       s));
    *launches += 4;
    // K2: predecessor DAG in CSR-by-source
    BCK(outdeg.alloc(8 * (n_nets + 1)));
    BCK(indeg.alloc(4 * n_nets));
    BCK(cudaMemsetAsync(outdeg.p, 0, 8 * (n_nets + 1), s));
    BCK(cudaMemsetAsync(indeg.p, 0, 4 * n_nets, s));
    DevBuf od32;
    BCK(od32.alloc(4 * (n_nets + 1)));
    BCK(cudaMemsetAsync(od32.p, 0, 4 * (n_nets + 1), s));
    k_edges_count<<<nblk(n_keys, 256), 256, 0, s>>>(kout.as<uint64_t>(), n_keys, od32.as<int32_t>(),
                                                     indeg.as<int32_t>());
    BCK(cudaGetLastError());
    // widen to int64 and scan
    k_widen<<<nblk(n_nets + 1, 256), 256, 0, s>>>(od32.as<int32_t>(), outdeg.as<int64_t>(), n_nets + 1);
    BCK(cudaGetLastError());
    BCK(off.alloc(8 * (n_nets + 1)));
    BCK(cub::DeviceScan::ExclusiveSum(tmp.p, scan_bytes, outdeg.as<int64_t>(), off.as<int64_t>(), n_nets + 1, s));
    BCK(cursor.alloc(4 * n_nets));
    BCK(cudaMemsetAsync(cursor.p, 0, 4 * n_nets, s));
    int64_t n_edges = 0;
    BCK(cudaMemcpyAsync(&n_edges, off.as<int64_t>() + n_nets, 8, cudaMemcpyDeviceToHost, s));
    BCK(cudaStreamSynchronize(s));
    BCK(succ.alloc(4 * std::max<int64_t>(n_edges, 1)));
    k_edges_fill<<<nblk(n_keys, 256), 256, 0, s>>>(kout.as<uint64_t>(), n_keys, off.as<int64_t>(),
                                                    cursor.as<int32_t>(), succ.as<int32_t>());
    BCK(cudaGetLastError());
    *launches += 3;
    if (dag) {   // keep the DAG (Kahn below consumes indeg)
        dag->release();
        dag->n = n_nets;
        dag->n_edges = n_edges;
        BCK(dmalloc(&dag->off, 8 * (n_nets + 1)));
        BCK(dmalloc(&dag->succ, 4 * std::max<int64_t>(n_edges, 1)));
        BCK(dmalloc(&dag->indeg, 4 * n_nets));
        BCK(cudaMemcpyAsync(dag->off, off.p, 8 * (n_nets + 1), cudaMemcpyDeviceToDevice, s));
        BCK(cudaMemcpyAsync(dag->succ, succ.p, 4 * std::max<int64_t>(n_edges, 1), cudaMemcpyDeviceToDevice, s));
        BCK(cudaMemcpyAsync(dag->indeg, indeg.p, 4 * n_nets, cudaMemcpyDeviceToDevice, s));
    }
    // Kahn frontiers
    BCK(batch.alloc(4 * n_nets));
    BCK(fa.alloc(4 * n_nets));
    BCK(fb.alloc(4 * n_nets));
    BCK(cnt.alloc(8));
    BCK(cudaMemsetAsync(cnt.p, 0, 8, s));
    k_frontier0<<<nblk(n_nets, 256), 256, 0, s>>>(indeg.as<int32_t>(), n_nets, batch.as<int32_t>(),
                                                   fa.as<int32_t>(), cnt.as<int32_t>());
    BCK(cudaGetLastError());
    *launches += 1;
    int32_t nfront = 0;
    BCK(cudaMemcpyAsync(&nfront, cnt.p, 4, cudaMemcpyDeviceToHost, s));
    BCK(cudaStreamSynchronize(s));
    int32_t *cur = fa.as<int32_t>(), *nxt = fb.as<int32_t>();
    int32_t *dcount = cnt.as<int32_t>();
    int32_t round = 0;
    int64_t done = nfront;
    while (nfront > 0) {
        BCK(cudaMemsetAsync(dcount + 1, 0, 4, s));
        k_frontier_step<<<nblk(nfront, 128), 128, 0, s>>>(cur, nfront, off.as<int64_t>(), succ.as<int32_t>(),
                                                          indeg.as<int32_t>(), batch.as<int32_t>(), round, nxt,
                                                          dcount + 1);
        BCK(cudaGetLastError());
        *launches += 1;
        BCK(cudaMemcpyAsync(&nfront, dcount + 1, 4, cudaMemcpyDeviceToHost, s));
        BCK(cudaStreamSynchronize(s));
        done += nfront;
        std::swap(cur, nxt);
        round++;
    }
    if (done != n_nets) return cudaErrorUnknown;   // cannot happen: the DAG is ordered by rank
    n_batches = round;
    BCK(cudaMemcpyAsync(batch_of_rank.data(), batch.p, 4 * n_nets, cudaMemcpyDeviceToHost, s));
    BCK(cudaStreamSynchronize(s));
    return cudaSuccess;
}

cudaError_t gpu_dag_to_positions(DagDev &dag, const int64_t *h_rank_of_pos, int64_t **off_p, int32_t **succ_p,
                                 int32_t **indeg_p, cudaStream_t s, int64_t *launches) {
    const int64_t n = dag.n;
    *off_p = nullptr; *succ_p = nullptr; *indeg_p = nullptr;
    DevBuf rop, por, deg, tmp;
    BCK(rop.alloc(8 * std::max<int64_t>(n, 1)));
    BCK(por.alloc(4 * std::max<int64_t>(n, 1)));
    BCK(deg.alloc(8 * (n + 1)));
    BCK(dmalloc(off_p, 8 * (n + 1)));
    BCK(dmalloc(succ_p, 4 * std::max<int64_t>(dag.n_edges, 1)));
    BCK(dmalloc(indeg_p, 4 * std::max<int64_t>(n, 1)));
    if (n == 0) {
        BCK(cudaMemsetAsync(*off_p, 0, 8, s));
        return cudaStreamSynchronize(s);
    }
    BCK(cudaMemcpyAsync(rop.p, h_rank_of_pos, 8 * n, cudaMemcpyHostToDevice, s));
    BCK(cudaMemsetAsync(deg.p, 0, 8 * (n + 1), s));
    k_inverse<<<nblk(n, 256), 256, 0, s>>>(rop.as<int64_t>(), n, por.as<int32_t>());
    k_dag_deg<<<nblk(n, 256), 256, 0, s>>>(dag.off, dag.indeg, rop.as<int64_t>(), n, deg.as<int64_t>(), *indeg_p);
    BCK(cudaGetLastError());
    size_t scan_bytes = 0;
    BCK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, deg.as<int64_t>(), *off_p, n + 1, s));
    BCK(tmp.alloc(scan_bytes));
    BCK(cub::DeviceScan::ExclusiveSum(tmp.p, scan_bytes, deg.as<int64_t>(), *off_p, n + 1, s));
    k_dag_fill<<<nblk(n, 256), 256, 0, s>>>(dag.off, dag.succ, rop.as<int64_t>(), por.as<int32_t>(), *off_p, n,
                                             *succ_p);
    BCK(cudaGetLastError());
    *launches += 4;
    BCK(cudaStreamSynchronize(s));
    dag.release();
    return cudaSuccess;
}

}  // namespace gapla
