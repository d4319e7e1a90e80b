// CPU-only harness for the host tree builder of la_load_nets (no GPU needed): includes
// la_host.cpp and runs the same chunked, threaded Builder pass over a design's nets, timing it.
// Used to profile / tune the e2e path's largest host phase (tools/hostbench/run.py).
#define GAPLA_BUILD_PROF 1
#include "../../paper_2507_13375_b200/csrc/la_host.cpp"

#include <chrono>

extern "C" double gapla_bench_build(const la_net_desc *n, int X, int Y, int L, const uint8_t *dir,
                                    const uint8_t *routable, double r_avg, double W_D, double logit_k, double logit_b,
                                    double w_floor, int nthr_req, int64_t *out) {
    la_ctx *ctx = new la_ctx();   // leaked on purpose: its destructor talks to the CUDA runtime
    ctx->X = X; ctx->Y = Y; ctx->L = L;
    ctx->dir.assign(dir, dir + L);
    ctx->routable.assign(routable, routable + L);
    ctx->r_avg = r_avg; ctx->W_D = W_D; ctx->logit_k = logit_k; ctx->logit_b = logit_b; ctx->w_floor = w_floor;
    const int64_t N = n->n_nets;
    unsigned nthr = nthr_req > 0 ? (unsigned)nthr_req : std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(N, (int64_t)nthr * 8));
    std::vector<Chunk> chunks(nchunks);
    for (int64_t c = 0; c < nchunks; c++) {
        chunks[c].beg = N * c / nchunks;
        chunks[c].end = N * (c + 1) / nchunks;
    }
    auto t0 = std::chrono::steady_clock::now();
    std::atomic<int64_t> next{0};
    auto worker = [&]() {
        Builder B{ctx, n};
        for (int l = 0; l < ctx->L; l++) if (ctx->routable[l]) B.nlegal[ctx->dir[l]]++;
        for (;;) {
            int64_t c = next.fetch_add(1);
            if (c >= nchunks) break;
            Chunk &ch = chunks[c];
            reserve_chunk(ch, n);
            ch.node_off.assign(1, 0);
            ch.sink_off.assign(1, 0);
            ch.fp_off.assign(1, 0);
            for (int64_t net = ch.beg; net < ch.end; net++) {
                BuiltNet &a = ch.acc;
                std::string err = B.build(net, a);
                if (!err.empty()) { ch.err = err; ch.err_net = net; break; }
                ch.node_off.push_back((int64_t)a.xy.size());
                ch.sink_off.push_back((int64_t)a.p_layer.size());
                ch.fp_off.push_back((int64_t)a.fp.size());
                ch.max_height = std::max<int>(ch.max_height, B.last_height);
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned i = 1; i < nthr; i++) th.emplace_back(worker);
        worker();
        for (auto &t : th) t.join();
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    {   // the calling thread's section shares (single-thread runs: the whole build)
        uint64_t tot = 0;
        for (int k = 0; k < 12; k++) tot += bprof_acc[k];
        for (int k = 0; k < 12; k++)
            std::fprintf(stderr, "section %2d: %5.1f%%\n", k, tot ? 100.0 * bprof_acc[k] / tot : 0.0);
    }
    // checksums of the built forest (node count, sink count, footprint count, hash of every array)
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void *p, size_t bytes) {
        const unsigned char *b = (const unsigned char *)p;
        for (size_t i = 0; i < bytes; i++) { h ^= b[i]; h *= 1099511628211ull; }
    };
    int64_t nn = 0, ns = 0, nf = 0;
    for (auto &ch : chunks) {
        if (ch.err_net >= 0) { out[0] = -1; return secs; }
        const BuiltNet &a = ch.acc;
        nn += (int64_t)a.xy.size(); ns += (int64_t)a.p_layer.size(); nf += (int64_t)a.fp.size();
        mix(a.xy.data(), 4 * a.xy.size()); mix(a.kid.data(), 4 * a.kid.size()); mix(a.len.data(), 4 * a.len.size());
        mix(a.edir.data(), a.edir.size()); mix(a.nkid.data(), a.nkid.size()); mix(a.nl.data(), a.nl.size());
        mix(a.nh.data(), a.nh.size()); mix(a.sink0.data(), 4 * a.sink0.size()); mix(a.nsink.data(), 2 * a.nsink.size());
        mix(a.wd.data(), 8 * a.wd.size()); mix(a.ur.data(), 8 * a.ur.size()); mix(a.height.data(), 2 * a.height.size());
        mix(a.p_layer.data(), a.p_layer.size()); mix(a.p_cap.data(), 8 * a.p_cap.size()); mix(a.p_w.data(), 8 * a.p_w.size());
        mix(a.p_orig.data(), 8 * a.p_orig.size()); mix(a.fp.data(), 8 * a.fp.size());
        mix(&a.wl, 8); mix(&a.wsw, 8);
    }
    out[0] = nn; out[1] = ns; out[2] = nf; out[3] = (int64_t)h;
    return secs;
}
