// Internal declarations of the GAP-LA B200 library (host C++ <-> CUDA kernels).
// Not part of the ABI: include/la.h is.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/la.h"

namespace gapla {

constexpr int MAXL = 16;                      // layers supported by the kernels
constexpr int MAXKIDS = 4;                    // a GCell has 4 neighbours -> <= 4 children
constexpr int MAXPAIRS = MAXL * (MAXL + 1) / 2;
constexpr uint8_t NO_DIR = 255;               // edir of a root

// Small per-layer tables staged into shared memory by every kernel CTA.
struct TechTab {
    double r[MAXL], c[MAXL], vr[MAXL], ofw[MAXL];
    double VR[MAXL * MAXL];                   // VR[a][b] = sum_{k=min}^{max-1} vr[k], ascending k
};

// Device view of the grid state.  Demand state is packed: one int32 word per
// (unit edge or via cut, layer) = ((d - c) << 1) | (c == 0).  A commit adds 2.
// Wire H plane [y][x][h] (x < X-1, h = index among H layers), V plane
// [x][y][v] (y < Y-1): one straight run's words on all its legal layers are one
// contiguous block.  Via plane [y][x][k], k < L-1.
struct DevGrid {
    int32_t X, Y, L, LH, LV;
    int8_t lidx[MAXL];                        // index of layer l inside its direction plane
    uint8_t dir[MAXL], routable[MAXL];
    int32_t delta_lo, delta_hi;
    double W_D, W_CAP, W_CONG, W_VIA;
    int32_t *wH, *wV, *via;
    const double *Mpos, *Mzero;               // Eq. (3) marginal tables over [delta_lo, delta_hi]
    const TechTab *tab;
};

// Batch-major forest.  Nets of one conflict-free batch are contiguous; the
// nodes of one net are contiguous, ordered by height (leaves first, root last).
struct DevForest {
    int64_t n_nets, n_nodes, n_sinks;
    const uint32_t *xy;                       // x | y << 16
    const int32_t *kid;                       // [n_nodes][4] global child ids (E, W, N, S order), -1
    const int32_t *len;                       // parent-edge length (unit edges)
    const uint8_t *edir;                      // direction parent -> node (0 E, 1 W, 2 N, 3 S); NO_DIR at root
    const uint8_t *nkid, *nl, *nh;            // #children; lowest / highest pin layer (driver incl.); nl=255 if none
    const uint16_t *height;                   // height (leaves 0)
    const int32_t *sink0;                     // first sink (pin arrays) of the node
    const uint16_t *nsink;
    const double *wd, *ur;                    // W_D * w_n (Eq. 5), ur (O3)
    const uint8_t *p_layer;                   // sinks, grouped by node, input order
    const double *p_cap, *p_w;                // C_q; weight of the pin-via delay term
    const int64_t *p_orig;                    // input pin index
    const int64_t *net_node0;                 // [n_nets+1] first node of each net (batch-major)
    const int64_t *net_id;                    // input net index
    const uint8_t *net_pdrv;                  // driver pin layer
};

// Capacities of the warp-per-net (small) path of k_assign: a net whose LA tree
// has at most NS_MAX nodes and at most NP_MAX sinks keeps all its DP state in
// shared memory; larger nets take the CTA-per-net (big) path.
constexpr int NS_MAX = 32;
constexpr int NP_MAX = 64;
constexpr int ASSIGN_WARPS = 4;

struct DevScratch {
    // big-path DP state, indexed by (node - first node of the batch); sized for
    // the largest total node count of big nets in any batch
    double *bkap;                             // [.][L-1] ViaCong per cut
    double *bA, *bB, *bC;                     // [.][LD] O5 parent-edge terms by layer slot (bA holds S first)
    uint16_t *bchoice;                        // [.][LD] b | t << 8
    uint32_t *bentry;                         // [.][LD] son layers, byte i = son i
    double *froot;                            // [n_nets] f[root][p_drv]
    uint8_t *lay, *sb, *st;                   // decisions per node: entry layer, span (b, t)
    uint32_t *dec;                            // packed decisions for the multi-GPU reconcile
    double *Cd, *rcv, *Tin;                   // Elmore per node
    double *sink_delay, *net_cap, *net_rc;    // outputs (input order)
};

// Kernel launchers (la_kernels.cu).  All enqueue on `s`.
cudaError_t launch_pack_state(const DevGrid &G, const int32_t *wcap, const int32_t *wdem, const int32_t *vcap,
                              const int32_t *vdem, const int64_t *wire_off, cudaStream_t s);
cudaError_t launch_unpack_demand(const DevGrid &G, const int32_t *wcap, const int32_t *vcap, int32_t *wdem,
                                 int32_t *vdem, const int64_t *wire_off, cudaStream_t s);
struct AssignLaunch {
    int64_t net_beg, net_end;                 // nets of this launch (batch-major)
    int64_t nbig;                             // the first nbig of them take the big path
    int64_t node_base;                        // first node of the batch: base of the big-path scratch
    int32_t LD;                               // max(#H layers, #V layers): layer slots per direction
    int32_t MP;                               // max (entry layer, span bottom) tasks of one node
    int32_t commit;                           // fuse the demand commit (K8) into the kernel
};
size_t assign_smem_bytes(int L, int LD, int MP);
cudaError_t launch_assign(const DevGrid &G, const DevForest &F, const DevScratch &S, const AssignLaunch &a,
                          cudaStream_t s);
cudaError_t launch_commit(const DevGrid &G, const DevForest &F, const DevScratch &S, int64_t node_beg,
                          int64_t node_end, cudaStream_t s);
cudaError_t launch_pack_decisions(const DevScratch &S, int64_t node_beg, int64_t node_end, cudaStream_t s);
cudaError_t launch_unpack_decisions(const DevScratch &S, int64_t node_beg, int64_t node_end, cudaStream_t s);
cudaError_t launch_elmore(const DevGrid &G, const DevForest &F, const DevScratch &S, int64_t net_beg,
                          int64_t net_end, cudaStream_t s);

// GPU conflict-free batching (la_batch.cu): keys = (element << 32) | rank,
// returns batch id per rank (host vector) and the number of batches.
cudaError_t gpu_conflict_batches(const uint64_t *h_keys, int64_t n_keys, int elem_bits, int64_t n_nets,
                                 std::vector<int32_t> &batch_of_rank, int32_t &n_batches, cudaStream_t s,
                                 int64_t *launches);

}  // namespace gapla
