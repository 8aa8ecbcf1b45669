// engine.cpp -- host orchestration of the Step-1 GPU path and the C ABI
// (include/labs_gpu.h).  Replaces run_saw_pool (saw.cpp:218-267): walks are
// enumerated in the reference's --threads 1 order (walker, restart), generated
// and run on the GPU in batches, and their sieve hits are replayed on the host
// through DedupSink -> CountingSink semantics (candidate.hpp:84-99,
// saw.cpp:173-194) before reaching the caller's sink.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "host_util.hpp"

namespace labs_b200 {

cudaError_t launch_saw_walk(const WalkParams& P, int grid, cudaStream_t st, int* score_out,
                            int* corr_out);
cudaError_t launch_saw_seed(const SeedParams& P, cudaStream_t st);
int walk_blocks_per_sm(WalkParams& P);  // (also places the fm table)

namespace {
thread_local std::string g_error;
}
void set_error(const std::string& msg) { g_error = msg; }

#define LABS_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess) {                                                           \
            throw CudaFailure(std::string(#call) + ": " + cudaGetErrorString(_e));         \
        }                                                                                  \
    } while (0)

struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void reserve(size_t count) {
        if (count <= n) return;
        release();
        LABS_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
    }
};

// Grow-only pinned host staging (async D2H drains of the record buffer and walk stats).
template <typename T>
struct PinnedBuf {
    T* p = nullptr;
    size_t n = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
    void reserve(size_t count) {
        if (count <= n) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        LABS_CUDA(cudaMallocHost(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
    }
};

// One restart range of one walker, in --threads 1 order.
struct Segment {
    uint32_t walker;
    int64_t r0, r1;
};

struct WalkRecordView {
    int64_t walk;        // batch-local walk index
    int64_t iteration;
    int64_t energy;
    uint64_t hash;       // canonical_hash(0) of the full sequence (computed on the device)
    const uint32_t* half;
};

struct BatchOut {
    std::vector<uint32_t> rec;    // count x rec_words
    int64_t nrec = 0;
    std::vector<int64_t> stats;   // nwalks x kWalkStatWords
    std::vector<int64_t> walk_walker, walk_restart;  // per batch walk
    double kernel_ms = 0, seed_ms = 0;
    int64_t h2d = 0, d2h = 0;  // bytes copied for this batch
};

// Per-device state: stream, events, uploaded tables, batch buffers.
class DeviceRunner {
public:
    int dev = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev[4] = {};
    WalkParams wp{};
    int grid_cap = 0;
    DevBuf<uint64_t> fm, tab, tabfull, rng;
    DevBuf<uint32_t> halves, rec, seg_walker, seg_prefix;
    DevBuf<int64_t> stats, seg_rest, seg_off;
    DevBuf<int32_t> seg_init;
    DevBuf<unsigned long long> rec_count;
    PinnedBuf<uint32_t> h_rec;
    PinnedBuf<int64_t> h_stats;
    PinnedBuf<unsigned long long> h_count;
    int64_t rec_cap = 0;

    ~DeviceRunner() {
        if (st) {
            cudaSetDevice(dev);
            for (auto& e : ev)
                if (e) cudaEventDestroy(e);
            cudaStreamDestroy(st);
        }
    }

    void init(int device, const WalkParams& params) {
        dev = device;
        wp = params;
        LABS_CUDA(cudaSetDevice(dev));
        LABS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        for (auto& e : ev) LABS_CUDA(cudaEventCreate(&e));
        const auto& tt = TabTables::get();
        const int kp1 = wp.kp1, L = wp.L;
        std::vector<uint64_t> hfm(3 * static_cast<size_t>(kp1));
        std::vector<uint64_t> htab(4 * static_cast<size_t>(kp1));
        std::vector<uint64_t> hfull(2 * static_cast<size_t>(L));
        for (int t = 0; t < 2; ++t)
            for (int i = 0; i < kp1; ++i) {
                hfm[static_cast<size_t>(t) * kp1 + i] = tt.t[t][i][0] ^ tt.t[t][i][1];
                htab[(static_cast<size_t>(t) * kp1 + i) * 2 + 0] = tt.t[t][i][0];
                htab[(static_cast<size_t>(t) * kp1 + i) * 2 + 1] = tt.t[t][i][1];
            }
        for (int j = 0; j < L; ++j) {
            hfull[2 * static_cast<size_t>(j)] = tt.t[0][j][0];
            hfull[2 * static_cast<size_t>(j) + 1] = tt.t[0][j][1];
        }
        for (int j = 0; j < kp1; ++j) {  // a skew flip at half index j toggles j and L-1-j
            uint64_t m = tt.t[0][j][0] ^ tt.t[0][j][1];
            if (L - 1 - j != j) m ^= tt.t[0][L - 1 - j][0] ^ tt.t[0][L - 1 - j][1];
            hfm[2 * static_cast<size_t>(kp1) + j] = m;
        }
        fm.reserve(hfm.size());
        tab.reserve(htab.size());
        tabfull.reserve(hfull.size());
        LABS_CUDA(cudaMemcpyAsync(fm.p, hfm.data(), hfm.size() * 8, cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaMemcpyAsync(tab.p, htab.data(), htab.size() * 8, cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaMemcpyAsync(tabfull.p, hfull.data(), hfull.size() * 8, cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaStreamSynchronize(st));  // host staging vectors die at scope end
        wp.fm = fm.p;
        wp.tab = tab.p;
        wp.tabfull = tabfull.p;
        wp.salt0 = tt.salt[0][kp1];
        wp.salt1 = tt.salt[1][kp1];
        wp.salt_full = tt.salt[0][L];
        int sms = 0;
        LABS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int bps = std::max(1, walk_blocks_per_sm(wp));
        grid_cap = sms * bps;
        rec_count.reserve(2);  // [0] records emitted, [1] the kernel's walk-group queue
    }

    // Generate halves for the segments on the device (K3).
    void seed(const std::vector<Segment>& segs, const Derived& d, uint64_t seed,
              std::vector<std::array<uint64_t, 4>>& states, const std::vector<int32_t>& init,
              int64_t nwalks, BatchOut& out) {
        const int nseg = static_cast<int>(segs.size());
        std::vector<uint32_t> hw(nseg), hp(nseg);
        std::vector<int64_t> hr(nseg), ho(nseg);
        std::vector<uint64_t> hs(4 * static_cast<size_t>(nseg));
        int64_t off = 0;
        for (int i = 0; i < nseg; ++i) {
            hw[i] = segs[i].walker;
            hp[i] = d.prefix_bits[segs[i].walker % static_cast<uint32_t>(d.nprefix)];
            hr[i] = segs[i].r1 - segs[i].r0;
            ho[i] = off;
            off += hr[i];
            for (int j = 0; j < 4; ++j) hs[4 * static_cast<size_t>(i) + j] = states[i][j];
        }
        seg_walker.reserve(nseg);
        seg_prefix.reserve(nseg);
        seg_rest.reserve(nseg);
        seg_off.reserve(nseg);
        seg_init.reserve(nseg);
        rng.reserve(4 * static_cast<size_t>(nseg));
        halves.reserve(static_cast<size_t>(nwalks) * wp.hw);
        LABS_CUDA(cudaMemcpyAsync(seg_walker.p, hw.data(), 4 * nseg, cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaMemcpyAsync(seg_prefix.p, hp.data(), 4 * nseg, cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaMemcpyAsync(seg_rest.p, hr.data(), 8 * nseg, cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaMemcpyAsync(seg_off.p, ho.data(), 8 * nseg, cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaMemcpyAsync(seg_init.p, init.data(), 4 * nseg, cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaMemcpyAsync(rng.p, hs.data(), 32 * static_cast<size_t>(nseg),
                                  cudaMemcpyHostToDevice, st));
        out.h2d += static_cast<int64_t>(nseg) * (4 + 4 + 8 + 8 + 4 + 32);
        SeedParams sp{};
        sp.kp1 = wp.kp1;
        sp.p = wp.p;
        sp.hw = wp.hw;
        sp.nseg = nseg;
        sp.seed = seed;
        sp.walker_ids = seg_walker.p;
        sp.prefix_bits = seg_prefix.p;
        sp.seg_restarts = seg_rest.p;
        sp.seg_offset = seg_off.p;
        sp.seg_init = seg_init.p;
        sp.rng_state = rng.p;
        sp.halves = halves.p;
        LABS_CUDA(cudaEventRecord(ev[2], st));
        LABS_CUDA(launch_saw_seed(sp, st));
        LABS_CUDA(cudaEventRecord(ev[3], st));
        LABS_CUDA(cudaMemcpyAsync(hs.data(), rng.p, 32 * static_cast<size_t>(nseg),
                                  cudaMemcpyDeviceToHost, st));
        LABS_CUDA(cudaStreamSynchronize(st));
        out.d2h += 32 * static_cast<int64_t>(nseg);
        float ms = 0;
        LABS_CUDA(cudaEventElapsedTime(&ms, ev[2], ev[3]));
        out.seed_ms += ms;
        for (int i = 0; i < nseg; ++i)
            for (int j = 0; j < 4; ++j) states[i][j] = hs[4 * static_cast<size_t>(i) + j];
    }

    void upload_halves(const std::vector<uint32_t>& h, int64_t nwalks) {
        halves.reserve(static_cast<size_t>(nwalks) * wp.hw);
        LABS_CUDA(cudaMemcpyAsync(halves.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st));
    }

    // Run K1 over `nwalks` walks whose halves are resident; copy back records + stats.
    void walk(int64_t nwalks, BatchOut& out, int* score_out = nullptr, int* corr_out = nullptr) {
        walk_launch(nwalks, score_out, corr_out);
        walk_finish(nwalks, out, score_out, corr_out);
    }

    // Enqueue K1 and the drains of the record count and the per-walk stats on this
    // runner's stream, without waiting (the pipelined pool overlaps the host replay of
    // the previous batch with it).
    // halves_at: the packed halves of these walks when they live elsewhere (the pipelined
    // pool seeds every batch at once into one runner's buffer); default: this runner's
    const uint32_t* halves_at = nullptr;
    void walk_launch(int64_t nwalks, int* score_out = nullptr, int* corr_out = nullptr) {
        stats.reserve(static_cast<size_t>(nwalks) * kWalkStatWords);
        if (rec_cap == 0) {
            rec_cap = std::max<int64_t>(1 << 16, 2 * nwalks);
            rec.reserve(static_cast<size_t>(rec_cap) * wp.rec_words);
        }
        WalkParams P = wp;
        P.nwalks = nwalks;
        P.halves = halves_at ? halves_at : halves.p;
        P.rec = rec.p;
        P.rec_cap = rec_cap;
        P.rec_count = rec_count.p;
        P.walk_next = rec_count.p + 1;
        P.walk_stats = stats.p;
        const int grid = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>(grid_cap, (nwalks + P.walks_per_block - 1) / P.walks_per_block)));
        LABS_CUDA(cudaMemsetAsync(rec_count.p, 0, 2 * sizeof(unsigned long long), st));
        LABS_CUDA(cudaEventRecord(ev[0], st));
        LABS_CUDA(launch_saw_walk(P, grid, st, score_out, corr_out));
        LABS_CUDA(cudaEventRecord(ev[1], st));
        h_count.reserve(1);
        LABS_CUDA(cudaMemcpyAsync(h_count.p, rec_count.p, sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, st));
        // the per-walk stats do not depend on the record count: drain them meanwhile
        h_stats.reserve(static_cast<size_t>(nwalks) * kWalkStatWords);
        LABS_CUDA(cudaMemcpyAsync(h_stats.p, stats.p,
                                  static_cast<size_t>(nwalks) * kWalkStatWords * 8,
                                  cudaMemcpyDeviceToHost, st));
    }

    // Wait for the launch, copy back records + stats; a record-buffer overflow grows the
    // buffer and reruns the (deterministic) walks.
    void walk_finish(int64_t nwalks, BatchOut& out, int* score_out = nullptr, int* corr_out = nullptr) {
        for (int attempt = 0; attempt < 3; ++attempt) {
            if (attempt > 0) walk_launch(nwalks, score_out, corr_out);
            LABS_CUDA(cudaStreamSynchronize(st));
            const unsigned long long cnt = *h_count.p;
            float ms = 0;
            LABS_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
            out.kernel_ms += ms;
            if (static_cast<int64_t>(cnt) > rec_cap) {  // overflow: grow and rerun (deterministic)
                rec_cap = static_cast<int64_t>(cnt) + cnt / 4 + 1024;
                rec.reserve(static_cast<size_t>(rec_cap) * wp.rec_words);
                continue;
            }
            out.nrec = static_cast<int64_t>(cnt);
            out.rec.resize(static_cast<size_t>(cnt) * wp.rec_words);
            out.stats.resize(static_cast<size_t>(nwalks) * kWalkStatWords);
            if (cnt) {
                h_rec.reserve(out.rec.size());
                LABS_CUDA(cudaMemcpyAsync(h_rec.p, rec.p, out.rec.size() * 4,
                                          cudaMemcpyDeviceToHost, st));
                LABS_CUDA(cudaStreamSynchronize(st));
                std::memcpy(out.rec.data(), h_rec.p, out.rec.size() * 4);
            }
            std::memcpy(out.stats.data(), h_stats.p, out.stats.size() * 8);
            out.d2h += static_cast<int64_t>(sizeof cnt + out.rec.size() * 4 + out.stats.size() * 8);
            return;
        }
        throw CudaFailure("record buffer overflow persisted");
    }
};

// Device contexts (stream, events, uploaded hash tables, grow-only batch buffers) are kept
// across run_saw_pool calls with the same walk geometry, so a call pays no allocation or
// table upload when the configuration repeats (the pipeline calls Step 1 once per round).
// (heap-allocated and never destroyed: no CUDA calls from static destructors at exit)
std::mutex g_runner_mu;
std::vector<std::unique_ptr<DeviceRunner>>& g_runner_pool = *new std::vector<std::unique_ptr<DeviceRunner>>();

bool same_geometry(const WalkParams& a, const WalkParams& b) {
    return a.L == b.L && a.p == b.p && a.t_i == b.t_i && a.bloom_bits == b.bloom_bits &&
           a.bloom_k == b.bloom_k && a.count_visited == b.count_visited &&
           a.debug_check == b.debug_check && a.lpw == b.lpw && a.R == b.R;  // (LABS_LPW)
}

std::unique_ptr<DeviceRunner> acquire_runner(int dev, const WalkParams& wp) {
    {
        std::lock_guard<std::mutex> lock(g_runner_mu);
        for (size_t i = 0; i < g_runner_pool.size(); ++i)
            if (g_runner_pool[i]->dev == dev && same_geometry(g_runner_pool[i]->wp, wp)) {
                std::unique_ptr<DeviceRunner> r = std::move(g_runner_pool[i]);
                g_runner_pool.erase(g_runner_pool.begin() + static_cast<long>(i));
                r->wp.e_l = wp.e_l;
                return r;
            }
    }
    std::unique_ptr<DeviceRunner> r(new DeviceRunner());
    r->init(dev, wp);
    return r;
}

void release_runners(std::vector<std::unique_ptr<DeviceRunner>>& rs) {
    std::lock_guard<std::mutex> lock(g_runner_mu);
    for (auto& r : rs)
        if (r && g_runner_pool.size() < 16) g_runner_pool.push_back(std::move(r));
    rs.clear();
}

int device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

std::string walk_params_for(const Derived& d, bool count_visited, bool debug, WalkParams& wp) {
    std::string err = make_walk_params(d.L, d.p, d.t_i, d.e_l, d.bloom_bits, d.bloom_k, wp);
    wp.count_visited = count_visited ? 1 : 0;
    wp.debug_check = debug ? 1 : 0;
    return err;
}

// Record views of a batch sorted by (walk, iteration); `start[w]..start[w+1]` indexes walk w.
struct GroupedRecords {
    std::vector<WalkRecordView> recs;
    std::vector<int64_t> start;
    const WalkRecordView* begin(int64_t w) const { return recs.data() + start[static_cast<size_t>(w)]; }
    const WalkRecordView* end(int64_t w) const { return recs.data() + start[static_cast<size_t>(w) + 1]; }
};

GroupedRecords group_records(const BatchOut& b, int rec_words, int64_t nwalks) {
    GroupedRecords g;
    g.recs.resize(static_cast<size_t>(b.nrec));
    g.start.assign(static_cast<size_t>(nwalks) + 1, 0);
    for (int64_t i = 0; i < b.nrec; ++i) {
        const uint32_t* r = &b.rec[static_cast<size_t>(i) * rec_words];
        g.recs[static_cast<size_t>(i)] = WalkRecordView{
            static_cast<int64_t>(r[0]), static_cast<int64_t>(r[1]),
            static_cast<int64_t>(static_cast<int32_t>(r[2])),
            static_cast<uint64_t>(r[4]) | (static_cast<uint64_t>(r[5]) << 32), r + kRecHeader};
        ++g.start[static_cast<size_t>(r[0]) + 1];
    }
    std::sort(g.recs.begin(), g.recs.end(), [](const WalkRecordView& a, const WalkRecordView& c) {
        return a.walk != c.walk ? a.walk < c.walk : a.iteration < c.iteration;
    });
    for (int64_t w = 0; w < nwalks; ++w) g.start[static_cast<size_t>(w) + 1] += g.start[static_cast<size_t>(w)];
    return g;
}

void half_bits_to_signs(const uint32_t* bits, int kp1, int8_t* half) {
    for (int i = 0; i < kp1; ++i) half[i] = ((bits[i >> 5] >> (i & 31)) & 1) ? 1 : -1;
}

// Host replay of one walk's sieve hits: DedupSink -> CountingSink -> user sink.
// Dedup uses the device-computed canonical_hash(0); only delivered candidates are expanded.
// Delivery is per candidate (`emit`) or in batches (`emit_batch`, flushed every kBatch).
struct SinkChain {
    static constexpr int kBatch = 8192;
    const labs_saw_config* cfg;
    const Derived* d;
    labs_candidate_fn emit;
    labs_candidate_batch_fn emit_batch;
    void* user;
    std::unordered_set<uint64_t> seen;
    int64_t emitted = 0;
    bool stop = false;
    bool aborted = false;
    std::vector<int8_t> half, full;
    // pending batch: accepted records (half bits still packed), expanded at flush
    std::vector<const uint32_t*> b_half;
    std::vector<int8_t> b_signs;
    std::vector<int64_t> b_energy, b_walker, b_restart, b_iter;
    std::vector<int32_t> b_class;
    // full position j of the skew expansion (skew.cpp:14-26) reads half bit src[j], negated
    // when neg[j]
    std::vector<int16_t> x_src;
    std::vector<uint8_t> x_neg;

    void deliver(uint32_t walker, int64_t restart, const WalkRecordView& r) {
        if (!seen.insert(r.hash).second) return;
        const int64_t n = ++emitted;
        if (cfg->candidate_quota > 0) {
            if (n > cfg->candidate_quota) {
                stop = true;
                --emitted;
                return;
            }
            if (n >= cfg->candidate_quota) stop = true;
        }
        if (aborted) return;
        const int cls = static_cast<int>(walker % static_cast<uint32_t>(d->nprefix));
        if (emit_batch) {
            b_half.push_back(r.half);
            b_energy.push_back(r.energy);
            b_walker.push_back(walker);
            b_restart.push_back(restart);
            b_iter.push_back(r.iteration);
            b_class.push_back(cls);
            if (static_cast<int>(b_energy.size()) >= kBatch) flush();
            return;
        }
        if (emit) {
            half.resize(static_cast<size_t>(d->kp1));
            full.resize(static_cast<size_t>(d->L));
            half_bits_to_signs(r.half, d->kp1, half.data());
            expand_skew(half.data(), d->kp1, full.data());
            labs_candidate c{};
            c.length = d->L;
            c.origin = 0;
            c.energy = r.energy;
            c.signs = full.data();
            c.prefix = d->p > 0 ? &d->prefixes[static_cast<size_t>(cls) * d->p] : nullptr;
            c.prefix_len = d->p;
            c.walker = walker;
            c.restart = restart;
            c.iteration = r.iteration;
            if (emit(user, &c) != 0) aborted = true;
        }
    }

    void expand_range(size_t i0, size_t i1) {
        const int L = d->L;
        for (size_t i = i0; i < i1; ++i) {
            const uint32_t* bits = b_half[i];
            int8_t* out = b_signs.data() + i * static_cast<size_t>(L);
            for (int j = 0; j < L; ++j) {
                const int src = x_src[static_cast<size_t>(j)];
                const int bit = static_cast<int>((bits[src >> 5] >> (src & 31)) & 1u) ^ x_neg[static_cast<size_t>(j)];
                out[j] = bit ? 1 : -1;
            }
        }
    }

    // Expands the pending records (in parallel for large batches; the order and the
    // dedup decisions were fixed in deliver) and hands them to emit_batch.  Must run
    // before the records' batch buffer is released.
    void flush() {
        if (!emit_batch || b_energy.empty() || aborted) {
            b_half.clear();
            b_energy.clear(), b_walker.clear(), b_restart.clear(), b_iter.clear(), b_class.clear();
            return;
        }
        const int L = d->L, k = d->k;
        if (static_cast<int>(x_src.size()) != L) {
            x_src.resize(static_cast<size_t>(L));
            x_neg.resize(static_cast<size_t>(L));
            for (int j = 0; j < L; ++j) {
                const int i = j > k ? j - k : 0;
                x_src[static_cast<size_t>(j)] = static_cast<int16_t>(j > k ? k - i : j);
                x_neg[static_cast<size_t>(j)] = static_cast<uint8_t>(i & 1);
            }
        }
        const size_t n = b_energy.size();
        b_signs.resize(n * static_cast<size_t>(L));
        const size_t nthreads = std::min<size_t>(
            n / 1024, std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
        if (nthreads <= 1) {
            expand_range(0, n);
        } else {
            std::vector<std::thread> th;
            const size_t chunk = (n + nthreads - 1) / nthreads;
            for (size_t t = 0; t < nthreads; ++t)
                th.emplace_back([this, t, chunk, n] {
                    expand_range(t * chunk, std::min(n, (t + 1) * chunk));
                });
            for (auto& x : th) x.join();
        }
        labs_candidate_batch b{};
        b.count = static_cast<int32_t>(n);
        b.length = L;
        b.prefix_len = d->p;
        b.origin = 0;
        b.signs = b_signs.data();
        b.energy = b_energy.data();
        b.walker = b_walker.data();
        b.restart = b_restart.data();
        b.iteration = b_iter.data();
        b.prefix_class = b_class.data();
        b.prefixes = d->p > 0 ? d->prefixes.data() : nullptr;
        if (emit_batch(user, &b) != 0) aborted = true;
        b_half.clear();
        b_energy.clear(), b_walker.clear(), b_restart.clear(), b_iter.clear(), b_class.clear();
    }
};

struct PoolAccum {
    labs_pool_stats st{};
    bool best_set = false;
    int64_t diverged = 0;
};

// Walker list of this call: [walker_begin, walker_end) filtered by class shard.
std::vector<uint32_t> walker_list(const labs_saw_config& cfg, const Derived& d, int shard_index,
                                  int shard_count) {
    std::vector<uint32_t> out;
    const int w0 = std::max(0, cfg.walker_begin);
    const int w1 = cfg.walker_end > 0 ? std::min(cfg.walker_end, cfg.walkers) : cfg.walkers;
    for (int w = w0; w < w1; ++w) {
        const int cls = w % d.nprefix;
        if (shard_count > 1 && cls % shard_count != shard_index) continue;
        out.push_back(static_cast<uint32_t>(w));
    }
    return out;
}

constexpr int64_t kMaxBatchWalks = 1 << 20;
constexpr int64_t kPipelineBatches = 8;  // single-device pool: batches per call (at least 2 waves each)

int pool_run(const labs_saw_config& cfg, labs_candidate_fn emit, labs_candidate_batch_fn emit_batch,
             void* user, labs_pool_stats* out) {
    const auto t0 = std::chrono::steady_clock::now();
    Derived d;
    std::string err = derive(cfg, d);
    if (!err.empty()) {
        set_error(err);
        return LABS_EINVAL;
    }
    WalkParams wp;
    err = walk_params_for(d, cfg.count_visited != 0, cfg.debug_check_energy != 0, wp);
    if (!err.empty()) {
        set_error(err);
        return LABS_EINVAL;
    }
    const int ndev_avail = device_count();
    if (ndev_avail <= 0) {
        set_error("no CUDA device available (the Step-1 engine has no CPU fallback)");
        return LABS_ENODEV;
    }
    const int first = std::max(0, cfg.device);
    // n_gpus class shards run concurrently, shard g on device first + g (mod the devices
    // available from `first`); more shards than devices share a device (separate streams)
    const int ngpu = std::max(1, cfg.n_gpus);
    const int ndev_use = std::max(1, ndev_avail - first);
    if (first >= ndev_avail) {
        set_error("device ordinal out of range");
        return LABS_ENODEV;
    }
    const int sidx = cfg.shard_count > 1 ? cfg.shard_index : 0;
    const int scnt = cfg.shard_count > 1 ? cfg.shard_count : 1;
    const std::vector<uint32_t> walkers = walker_list(cfg, d, sidx, scnt);
    const bool coupled = cfg.candidate_quota > 0 || cfg.stop_at_energy > 0 ||
                         cfg.time_budget_s > 0 || cfg.max_restarts == 0;

    PoolAccum acc;
    SinkChain sink{};
    sink.cfg = &cfg;
    sink.d = &d;
    sink.emit = emit;
    sink.emit_batch = emit_batch;
    sink.user = user;
    std::vector<std::unique_ptr<DeviceRunner>> runners;
    try {
        for (int g = 0; g < (coupled ? 1 : ngpu); ++g)
            runners.push_back(acquire_runner(first + g % ndev_use, wp));
        // ---- build the ordered walk sequence as batches of segments ----
        // Per walker: state carried across batches (only in coupled mode can a walker's
        // restarts span batches).
        const auto deadline_hit = [&]() {
            return cfg.time_budget_s > 0 &&
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() >=
                       cfg.time_budget_s;
        };
        auto process_batch = [&](const std::vector<Segment>& segs, BatchOut& b) {
            const int64_t nw = static_cast<int64_t>(b.walk_walker.size());
            const auto groups = group_records(b, wp.rec_words, nw);
            for (int64_t i = 0; i < nw && !sink.stop && !sink.aborted; ++i) {
                const int64_t* s = &b.stats[static_cast<size_t>(i) * kWalkStatWords];
                for (const WalkRecordView* r = groups.begin(i); r != groups.end(i); ++r)
                    sink.deliver(static_cast<uint32_t>(b.walk_walker[i]), b.walk_restart[i], *r);
                ++acc.st.walks;
                acc.st.iterations += s[kWsIterations];
                acc.st.emitted_raw += s[kWsEmitted];
                acc.st.delta_evals += s[kWsDeltaEvals] >= 0 ? s[kWsDeltaEvals] : 0;
                acc.st.exhausted_walks += s[kWsExhausted];
                acc.st.wide_iterations += s[kWsWideIters];
                acc.diverged += s[kWsDiverged];
                // offer_best (saw.cpp:160-169)
                if (!acc.best_set || s[kWsBest] < acc.st.best_energy) {
                    acc.st.best_energy = s[kWsBest];
                    acc.best_set = true;
                    if (cfg.stop_at_energy > 0 && s[kWsBest] <= cfg.stop_at_energy) sink.stop = true;
                }
                if (acc.diverged) break;
            }
            sink.flush();  // the batch's record buffer dies with `b`
            (void)segs;
        };

        if (!coupled) {
            // Every (walker, restart) walk is independent: split walkers across GPUs by
            // restriction class, run each GPU's list in batches, merge in walker order.
            const int64_t R = cfg.max_restarts;
            std::vector<std::vector<uint32_t>> per_dev(static_cast<size_t>(ngpu));
            for (uint32_t w : walkers)
                per_dev[static_cast<size_t>((w % static_cast<uint32_t>(d.nprefix)) % ngpu)].push_back(w);
            std::vector<std::vector<BatchOut>> outs(static_cast<size_t>(ngpu));
            std::vector<std::vector<std::vector<Segment>>> segs_all(static_cast<size_t>(ngpu));
            std::vector<std::string> errs(static_cast<size_t>(ngpu));
            // batches: whole walkers while they fit, else restart ranges
            const auto make_batches = [&](const std::vector<uint32_t>& wl, int64_t max_walks) {
                std::vector<std::vector<Segment>> batches;
                std::vector<Segment> cur;
                int64_t cur_walks = 0;
                for (uint32_t w : wl) {
                    int64_t r = 0;
                    while (r < R) {
                        const int64_t take = std::min(R - r, max_walks - cur_walks);
                        cur.push_back(Segment{w, r, r + take});
                        cur_walks += take;
                        r += take;
                        if (cur_walks == max_walks) {
                            batches.push_back(std::move(cur));
                            cur.clear();
                            cur_walks = 0;
                        }
                    }
                }
                if (!cur.empty()) batches.push_back(std::move(cur));
                return batches;
            };
            // Seed one batch on `dr` (K3); a walker split across batches continues from the
            // generator state its previous batch ended with.
            struct Carry {
                uint32_t walker = 0xffffffffu;
                std::array<uint64_t, 4> state{};
            };
            const auto seed_batch = [&](DeviceRunner& dr, const std::vector<Segment>& segs, Carry& carry,
                                        BatchOut& b) {
                std::vector<std::array<uint64_t, 4>> states(segs.size());
                std::vector<int32_t> init(segs.size(), 1);
                int64_t nw = 0;
                for (size_t i = 0; i < segs.size(); ++i) {
                    if (segs[i].r0 > 0 && segs[i].walker == carry.walker) {
                        init[i] = 0;
                        states[i] = carry.state;
                    }
                    for (int64_t r = segs[i].r0; r < segs[i].r1; ++r) {
                        b.walk_walker.push_back(segs[i].walker);
                        b.walk_restart.push_back(r);
                    }
                    nw += segs[i].r1 - segs[i].r0;
                }
                dr.seed(segs, d, cfg.seed, states, init, nw, b);
                carry.walker = segs.back().walker;
                carry.state = states.back();
                return nw;
            };
            auto dev_job = [&](int g) {
                try {
                    DeviceRunner& dr = *runners[static_cast<size_t>(g)];
                    LABS_CUDA(cudaSetDevice(dr.dev));
                    Carry carry;
                    for (auto& segs : make_batches(per_dev[static_cast<size_t>(g)], kMaxBatchWalks)) {
                        BatchOut b;
                        const auto tA = std::chrono::steady_clock::now();
                        const int64_t nw = seed_batch(dr, segs, carry, b);
                        const auto tB = std::chrono::steady_clock::now();
                        dr.walk(nw, b);
                        const auto tC = std::chrono::steady_clock::now();
                        if (std::getenv("LABS_TIMING"))
                            std::fprintf(stderr, "[labs] seed %.2f ms, walk+d2h %.2f ms (kernel %.2f)\n",
                                         std::chrono::duration<double, std::milli>(tB - tA).count(),
                                         std::chrono::duration<double, std::milli>(tC - tB).count(),
                                         b.kernel_ms);
                        outs[static_cast<size_t>(g)].push_back(std::move(b));
                        segs_all[static_cast<size_t>(g)].push_back(segs);
                    }
                } catch (const std::exception& e) {
                    errs[static_cast<size_t>(g)] = e.what();
                }
            };
            if (ngpu == 1) {
                // One device: the walks run as a pipeline of batches on two runners (two
                // streams and buffer sets).  While batch i runs -- and fills the SMs its
                // predecessor's tail leaves idle -- the host replays batch i-1 into the sink.
                runners.push_back(acquire_runner(first, wp));
                DeviceRunner* slot[2] = {runners[0].get(), runners[1].get()};
                LABS_CUDA(cudaSetDevice(slot[0]->dev));
                const int64_t resident = static_cast<int64_t>(slot[0]->grid_cap) * wp.walks_per_block;
                const int64_t total = static_cast<int64_t>(walkers.size()) * R;
                const char* nb_env = std::getenv("LABS_PIPELINE_BATCHES");  // (A/B knob)
                const int64_t nb = std::max<int64_t>(1, nb_env ? std::atoll(nb_env) : kPipelineBatches);
                const int64_t chunk = std::min<int64_t>(
                    kMaxBatchWalks, nb == 1 ? total : std::max<int64_t>(2 * resident, (total + nb - 1) / nb));
                const auto batches = make_batches(walkers, chunk);
                std::vector<BatchOut> bo(batches.size());
                std::vector<int64_t> nws(batches.size()), off(batches.size());
                // K3 once for the whole pool (walker order = batch order), so no batch waits on
                // a seed launch queued behind the other stream's walk kernel
                {
                    std::vector<Segment> all;
                    for (uint32_t w : walkers) all.push_back(Segment{w, 0, R});
                    std::vector<std::array<uint64_t, 4>> states(all.size());
                    std::vector<int32_t> init(all.size(), 1);
                    BatchOut sb;
                    slot[0]->seed(all, d, cfg.seed, states, init, total, sb);
                    acc.st.seed_ms += sb.seed_ms;
                    acc.st.h2d_bytes += sb.h2d;
                    acc.st.d2h_bytes += sb.d2h;
                }
                int64_t o = 0;
                for (size_t i = 0; i < batches.size(); ++i) {
                    off[i] = o;
                    nws[i] = 0;
                    for (const Segment& sg : batches[i]) {
                        for (int64_t r = sg.r0; r < sg.r1; ++r) {
                            bo[i].walk_walker.push_back(sg.walker);
                            bo[i].walk_restart.push_back(r);
                        }
                        nws[i] += sg.r1 - sg.r0;
                    }
                    o += nws[i];
                }
                const auto tD = std::chrono::steady_clock::now();
                double replay_ms = 0;
                const auto retire = [&](size_t j) {  // wait for batch j, replay it, free it
                    slot[j % 2]->walk_finish(nws[j], bo[j]);
                    acc.st.kernel_ms += bo[j].kernel_ms;
                    acc.st.seed_ms += bo[j].seed_ms;
                    acc.st.h2d_bytes += bo[j].h2d;
                    acc.st.d2h_bytes += bo[j].d2h;
                    const auto t = std::chrono::steady_clock::now();
                    if (!sink.aborted && acc.diverged == 0) process_batch(batches[j], bo[j]);
                    replay_ms += std::chrono::duration<double, std::milli>(
                        std::chrono::steady_clock::now() - t).count();
                    bo[j] = BatchOut();
                };
                size_t launched = 0, retired = 0;
                for (size_t i = 0; i < batches.size(); ++i) {
                    if (i >= 2) retire(retired++);  // batch i - 2: frees slot i % 2
                    if (sink.aborted || acc.diverged) break;
                    slot[i % 2]->halves_at = slot[0]->halves.p + static_cast<size_t>(off[i]) * wp.hw;
                    slot[i % 2]->walk_launch(nws[i]);
                    launched = i + 1;
                }
                while (retired < launched) retire(retired++);
                slot[0]->halves_at = slot[1]->halves_at = nullptr;
                if (std::getenv("LABS_TIMING"))
                    std::fprintf(stderr, "[labs] %zu pipelined batches of <= %lld walks: %.2f ms, "
                                 "host replay %.2f ms (overlapped)\n", batches.size(),
                                 static_cast<long long>(chunk),
                                 std::chrono::duration<double, std::milli>(
                                     std::chrono::steady_clock::now() - tD).count(), replay_ms);
            } else {
                std::vector<std::thread> th;
                for (int g = 0; g < ngpu; ++g) th.emplace_back(dev_job, g);
                for (auto& t : th) t.join();
            }
            for (const auto& e : errs)
                if (!e.empty()) throw CudaFailure(e);
            if (ngpu > 1) {
                for (int g = 0; g < ngpu; ++g) {  // device time = slowest device
                    double kms = 0, sms = 0;
                    for (const auto& b : outs[static_cast<size_t>(g)]) {
                        kms += b.kernel_ms;
                        sms += b.seed_ms;
                        acc.st.h2d_bytes += b.h2d;
                        acc.st.d2h_bytes += b.d2h;
                    }
                    acc.st.kernel_ms = std::max(acc.st.kernel_ms, kms);
                    acc.st.seed_ms = std::max(acc.st.seed_ms, sms);
                }
                // merge: walks of all devices in (walker, restart) order
                struct Ref {
                    uint32_t walker;
                    int64_t restart;
                    int g;
                    size_t b;
                    int64_t i;
                };
                std::vector<Ref> refs;
                std::vector<std::vector<GroupedRecords>> grp(static_cast<size_t>(ngpu));
                for (int g = 0; g < ngpu; ++g)
                    for (size_t bi = 0; bi < outs[static_cast<size_t>(g)].size(); ++bi) {
                        const BatchOut& b = outs[static_cast<size_t>(g)][bi];
                        grp[static_cast<size_t>(g)].push_back(
                            group_records(b, wp.rec_words, static_cast<int64_t>(b.walk_walker.size())));
                        for (size_t i = 0; i < b.walk_walker.size(); ++i)
                            refs.push_back(Ref{static_cast<uint32_t>(b.walk_walker[i]), b.walk_restart[i], g, bi,
                                               static_cast<int64_t>(i)});
                    }
                std::sort(refs.begin(), refs.end(), [](const Ref& a, const Ref& c) {
                    return a.walker != c.walker ? a.walker < c.walker : a.restart < c.restart;
                });
                for (const Ref& r : refs) {
                    const BatchOut& b = outs[static_cast<size_t>(r.g)][r.b];
                    const int64_t* s = &b.stats[static_cast<size_t>(r.i) * kWalkStatWords];
                    const GroupedRecords& gr = grp[static_cast<size_t>(r.g)][r.b];
                    for (const WalkRecordView* v = gr.begin(r.i); v != gr.end(r.i); ++v)
                        sink.deliver(r.walker, r.restart, *v);
                    ++acc.st.walks;
                    acc.st.iterations += s[kWsIterations];
                    acc.st.emitted_raw += s[kWsEmitted];
                    acc.st.delta_evals += s[kWsDeltaEvals] >= 0 ? s[kWsDeltaEvals] : 0;
                    acc.st.exhausted_walks += s[kWsExhausted];
                    acc.st.wide_iterations += s[kWsWideIters];
                    acc.diverged += s[kWsDiverged];
                    if (!acc.best_set || s[kWsBest] < acc.st.best_energy) {
                        acc.st.best_energy = s[kWsBest];
                        acc.best_set = true;
                    }
                }
                sink.flush();  // before the devices' record buffers are released
            }
        } else {
            // Coupled stop conditions: ordered batches, stop replay exactly like --threads 1.
            DeviceRunner& dr = *runners[0];
            int64_t batch_walks = 4096;
            size_t wi = 0;
            int64_t next_r = 0;
            std::array<uint64_t, 4> carry_state{};
            bool carry_valid = false;
            while (wi < walkers.size() && !sink.stop && !sink.aborted && acc.diverged == 0) {
                if (deadline_hit()) break;
                std::vector<Segment> segs;
                std::vector<std::array<uint64_t, 4>> states;
                std::vector<int32_t> init;
                BatchOut b;
                int64_t nw = 0;
                size_t wj = wi;
                int64_t r = next_r;
                while (nw < batch_walks && wj < walkers.size()) {
                    const int64_t lim = cfg.max_restarts > 0 ? cfg.max_restarts : INT64_MAX;
                    const int64_t take = std::min(lim - r, batch_walks - nw);
                    segs.push_back(Segment{walkers[wj], r, r + take});
                    states.push_back(carry_state);
                    init.push_back(r == 0 || !carry_valid ? 1 : 0);
                    for (int64_t q = r; q < r + take; ++q) {
                        b.walk_walker.push_back(walkers[wj]);
                        b.walk_restart.push_back(q);
                    }
                    nw += take;
                    r += take;
                    if (r >= lim) {
                        ++wj;
                        r = 0;
                        carry_valid = false;
                    }
                }
                dr.seed(segs, d, cfg.seed, states, init, nw, b);
                if (r > 0) {  // last walker continues in the next batch
                    carry_state = states.back();
                    carry_valid = true;
                }
                dr.walk(nw, b);
                acc.st.kernel_ms += b.kernel_ms;
                acc.st.seed_ms += b.seed_ms;
                acc.st.h2d_bytes += b.h2d;
                acc.st.d2h_bytes += b.d2h;
                process_batch(segs, b);
                wi = wj;
                next_r = r;
                batch_walks = std::min<int64_t>(batch_walks * 2, kMaxBatchWalks);
            }
        }
    } catch (const CudaFailure& e) {
        set_error(e.what());
        return LABS_ECUDA;  // runners dropped: their state may be unusable
    } catch (const std::bad_alloc&) {
        set_error("out of host memory");
        return LABS_ECUDA;
    }
    release_runners(runners);
    if (acc.diverged) {
        set_error("saw walk energy bookkeeping diverged");
        return LABS_ELOGIC;
    }
    sink.flush();
    acc.st.emitted = sink.emitted;
    acc.st.best_energy = acc.best_set ? acc.st.best_energy : 0;
    acc.st.delta_evals = cfg.count_visited ? acc.st.delta_evals : -1;
    int64_t free_bits = d.kp1 - d.p;
    acc.st.delta_evals_computed = (acc.st.iterations + acc.st.walks) * (free_bits > 0 ? free_bits : 0);
    acc.st.n_gpus = coupled ? 1 : ngpu;
    acc.st.wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (out) *out = acc.st;
    if (sink.aborted) {
        set_error("candidate sink aborted the run");
        return LABS_EABORT;
    }
    return LABS_OK;
}

// Seed-table mode on device 0.
int walks_from_halves(int L, int p, int64_t t_i, int64_t e_l, double fpr, const int8_t* halves,
                      int64_t nwalks, bool count, bool debug, labs_walk_result* res,
                      labs_record_fn on_rec, void* user, int64_t* deltas_out,
                      int64_t* corr_out, int64_t* energies_out) {
    if (L < 3 || L % 2 == 0) {
        set_error("length must be odd and >= 3");
        return LABS_EINVAL;
    }
    const int kp1 = (L + 1) / 2;
    if (p < 0 || p > kp1) {
        set_error("prefix length exceeds half length k+1");
        return LABS_EINVAL;
    }
    if (kp1 > kMaxHalf) {
        set_error("length exceeds the tabulation hash range");
        return LABS_EINVAL;
    }
    for (int64_t i = 0; i < nwalks * kp1; ++i)
        if (halves[i] != 1 && halves[i] != -1) {
            set_error("SkewHalf: elements must be +1 or -1");
            return LABS_EINVAL;
        }
    if (device_count() <= 0) {
        set_error("no CUDA device available (the Step-1 engine has no CPU fallback)");
        return LABS_ENODEV;
    }
    uint64_t bits;
    int bk;
    bloom_size(static_cast<uint64_t>(std::max<int64_t>(t_i, 1)) + 1, fpr, bits, bk);
    WalkParams wp;
    std::string err = make_walk_params(L, p, std::max<int64_t>(t_i, 1), e_l, bits, bk, wp);
    if (!err.empty()) {
        set_error(err);
        return LABS_EINVAL;
    }
    wp.t_i = t_i;
    wp.count_visited = count ? 1 : 0;
    wp.debug_check = debug ? 1 : 0;
    try {
        DeviceRunner dr;
        dr.init(0, wp);
        std::vector<uint32_t> hb(static_cast<size_t>(nwalks) * wp.hw, 0u);
        for (int64_t w = 0; w < nwalks; ++w)
            for (int i = 0; i < kp1; ++i)
                if (halves[w * kp1 + i] > 0) hb[static_cast<size_t>(w) * wp.hw + (i >> 5)] |= 1u << (i & 31);
        dr.upload_halves(hb, nwalks);
        BatchOut b;
        DevBuf<int> dscore, dcorr;
        if (deltas_out) {
            dscore.reserve(static_cast<size_t>(nwalks) * kp1);
            dcorr.reserve(static_cast<size_t>(nwalks) * std::max(1, kp1 - 1));
        }
        dr.walk(nwalks, b, deltas_out ? dscore.p : nullptr, deltas_out ? dcorr.p : nullptr);
        if (deltas_out) {
            std::vector<int> hs(static_cast<size_t>(nwalks) * kp1), hc(static_cast<size_t>(nwalks) * (kp1 - 1));
            LABS_CUDA(cudaMemcpy(hs.data(), dscore.p, hs.size() * 4, cudaMemcpyDeviceToHost));
            if (!hc.empty())
                LABS_CUDA(cudaMemcpy(hc.data(), dcorr.p, hc.size() * 4, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < hs.size(); ++i) deltas_out[i] = hs[i];
            if (corr_out)
                for (size_t i = 0; i < hc.size(); ++i) corr_out[i] = hc[i];
        }
        const auto groups = group_records(b, wp.rec_words, nwalks);
        std::vector<int8_t> half(static_cast<size_t>(kp1));
        for (int64_t w = 0; w < nwalks; ++w) {
            const int64_t* s = &b.stats[static_cast<size_t>(w) * kWalkStatWords];
            if (energies_out) energies_out[w] = s[kWsInitial];
            if (res) {
                labs_walk_result& r = res[w];
                r.iterations = s[kWsIterations];
                r.emitted = s[kWsEmitted];
                r.best_energy = s[kWsBest];
                r.initial_energy = s[kWsInitial];
                r.exhausted = s[kWsExhausted];
                r.delta_evals = s[kWsDeltaEvals];
                r.probe_rounds = s[kWsVisitedProbes];
                r.wide_iterations = s[kWsWideIters];
                r.diverged = s[kWsDiverged];
            }
            if (on_rec)
                for (const WalkRecordView* v = groups.begin(w); v != groups.end(w); ++v) {
                    half_bits_to_signs(v->half, kp1, half.data());
                    if (on_rec(user, w, v->iteration, v->energy, half.data(), kp1) != 0) return LABS_EABORT;
                }
        }
    } catch (const CudaFailure& e) {
        set_error(e.what());
        return LABS_ECUDA;
    }
    return LABS_OK;
}

// ---------------------------------------------------------------- bench plan
struct BenchPlan {
    labs_saw_config cfg;
    Derived d;
    std::unique_ptr<DeviceRunner> dr;
    DevBuf<uint8_t> l2_scratch;  // written before every rep: no rep starts with a warm L2
    static constexpr size_t kL2Flush = size_t(256) << 20;
    std::vector<Segment> segs;
    int64_t nwalks = 0;
};

}  // namespace labs_b200

// ============================================================================ C ABI
using namespace labs_b200;

struct labs_bench_plan {
    BenchPlan p;
};

extern "C" {

const char* labs_last_error(void) { return g_error.c_str(); }
const char* labs_version(void) { return "paper_2409_07222_b200 0.1 (sm_100a)"; }

uint64_t labs_canonical_hash(const int8_t* signs, int32_t n, int32_t table) {
    if (n < 0 || n > kMaxHalf || table < 0 || table > 1) return 0;
    return TabTables::get().hash(signs, n, table);
}

int labs_format_record(const int8_t* signs, int32_t n, int64_t energy, char* out, int32_t cap) {
    const std::string s = format_record(signs, n, energy);
    if (cap > 0) std::snprintf(out, static_cast<size_t>(cap), "%s", s.c_str());
    return static_cast<int>(s.size());
}

int labs_rank_prefixes(int32_t p, int8_t* out) {
    if (p < 1) {
        set_error("rank_prefixes: p must be >= 1");
        return LABS_EINVAL;
    }
    if (p > 30) {
        set_error("rank_prefixes: p > 30 is not enumerable");
        return LABS_EINVAL;
    }
    const auto v = rank_prefixes(p);
    std::copy(v.begin(), v.end(), out);
    return static_cast<int>(v.size() / static_cast<size_t>(p));
}

int labs_expand_skew(const int8_t* half, int32_t kp1, int8_t* full) {
    if (kp1 < 2) {
        set_error("SkewHalf: need k+1 >= 2 elements (L >= 3)");
        return LABS_EINVAL;
    }
    expand_skew(half, kp1, full);
    return LABS_OK;
}

int labs_device_count(int32_t* n) {
    *n = device_count();
    return LABS_OK;
}

int labs_saw_derive(const labs_saw_config* cfg, labs_saw_derived* out) {
    Derived d;
    std::string err = derive(*cfg, d);
    if (!err.empty()) {
        set_error(err);
        return LABS_EINVAL;
    }
    WalkParams wp;
    err = make_walk_params(d.L, d.p, d.t_i, d.e_l, d.bloom_bits, d.bloom_k, wp);
    out->prefix_len = d.p;
    out->bloom_hashes = d.bloom_k;
    out->iterations = d.t_i;
    out->energy_threshold = d.e_l;
    out->bloom_bits = d.bloom_bits;
    out->free_bits = d.kp1 - d.p;
    out->neighbours_per_lane = err.empty() ? wp.R : 0;
    if (!err.empty()) {
        set_error(err);
        return LABS_EINVAL;
    }
    return LABS_OK;
}

int labs_saw_pool_run(const labs_saw_config* cfg, labs_candidate_fn emit, void* user,
                      labs_pool_stats* stats) {
    if (!cfg) {
        set_error("null config");
        return LABS_EINVAL;
    }
    return pool_run(*cfg, emit, nullptr, user, stats);
}

int labs_saw_pool_run_batched(const labs_saw_config* cfg, labs_candidate_batch_fn emit, void* user,
                              labs_pool_stats* stats) {
    if (!cfg) {
        set_error("null config");
        return LABS_EINVAL;
    }
    return pool_run(*cfg, nullptr, emit, user, stats);
}

int labs_saw_walks(int32_t length, int32_t prefix_len, int64_t iterations,
                   int64_t energy_threshold, double bloom_fpr, const int8_t* halves,
                   int64_t nwalks, int32_t count_visited, int32_t debug_check,
                   labs_walk_result* results, labs_record_fn on_record, void* user) {
    if (iterations < 1) {
        set_error("saw: T_i must be >= 1");
        return LABS_EINVAL;
    }
    return walks_from_halves(length, prefix_len, iterations, energy_threshold, bloom_fpr, halves,
                             nwalks, count_visited != 0, debug_check != 0, results, on_record, user,
                             nullptr, nullptr, nullptr);
}

int labs_skew_flip_deltas(int32_t length, const int8_t* halves, int64_t nseq, int64_t* deltas,
                          int64_t* corr, int64_t* energies) {
    if (!deltas) {
        set_error("deltas output required");
        return LABS_EINVAL;
    }
    return walks_from_halves(length, 0, 1, 1, 0.5, halves, nseq, false, false, nullptr, nullptr,
                             nullptr, deltas, corr, energies);
}

int labs_bench_create(const labs_saw_config* cfg, labs_bench_plan** out) {
    auto* plan = new labs_bench_plan();
    BenchPlan& bp = plan->p;
    bp.cfg = *cfg;
    std::string err = derive(bp.cfg, bp.d);
    WalkParams wp;
    if (err.empty()) err = walk_params_for(bp.d, cfg->count_visited != 0, false, wp);
    if (err.empty() && cfg->max_restarts <= 0) err = "bench plan needs max_restarts > 0";
    if (!err.empty()) {
        delete plan;
        set_error(err);
        return LABS_EINVAL;
    }
    if (device_count() <= 0) {
        delete plan;
        set_error("no CUDA device available");
        return LABS_ENODEV;
    }
    try {
        bp.dr.reset(new DeviceRunner());
        bp.dr->init(std::max(0, cfg->device), wp);
        const int sidx = cfg->shard_count > 1 ? cfg->shard_index : 0;
        const int scnt = cfg->shard_count > 1 ? cfg->shard_count : 1;
        for (uint32_t w : walker_list(bp.cfg, bp.d, sidx, scnt))
            bp.segs.push_back(Segment{w, 0, cfg->max_restarts});
        bp.nwalks = static_cast<int64_t>(bp.segs.size()) * cfg->max_restarts;
        if (bp.nwalks > kMaxBatchWalks) throw CudaFailure("bench plan larger than one batch");
    } catch (const CudaFailure& e) {
        delete plan;
        set_error(e.what());
        return LABS_ECUDA;
    }
    *out = plan;
    return LABS_OK;
}

int labs_bench_run(labs_bench_plan* plan, int32_t reps, double* ms_per_rep, labs_pool_stats* last) {
    BenchPlan& bp = plan->p;
    try {
        DeviceRunner& dr = *bp.dr;
        LABS_CUDA(cudaSetDevice(dr.dev));
        double total = 0;
        BatchOut b;
        bp.l2_scratch.reserve(BenchPlan::kL2Flush);
        for (int r = 0; r < reps; ++r) {
            LABS_CUDA(cudaMemsetAsync(bp.l2_scratch.p, r & 0xff, BenchPlan::kL2Flush, dr.st));
            b = BatchOut();
            std::vector<std::array<uint64_t, 4>> states(bp.segs.size());
            std::vector<int32_t> init(bp.segs.size(), 1);
            dr.seed(bp.segs, bp.d, bp.cfg.seed, states, init, bp.nwalks, b);
            dr.walk(bp.nwalks, b);
            total += b.kernel_ms + b.seed_ms;
        }
        if (ms_per_rep) *ms_per_rep = reps > 0 ? total / reps : 0;
        if (last) {
            labs_pool_stats st{};
            st.walks = bp.nwalks;
            st.kernel_ms = b.kernel_ms;
            st.seed_ms = b.seed_ms;
            st.emitted_raw = b.nrec;
            for (int64_t i = 0; i < bp.nwalks; ++i) {
                const int64_t* s = &b.stats[static_cast<size_t>(i) * kWalkStatWords];
                st.iterations += s[kWsIterations];
                st.delta_evals += s[kWsDeltaEvals] >= 0 ? s[kWsDeltaEvals] : 0;
                st.exhausted_walks += s[kWsExhausted];
                st.wide_iterations += s[kWsWideIters];
                if (i == 0 || s[kWsBest] < st.best_energy) st.best_energy = s[kWsBest];
            }
            // post-dedup count of the last rep's sieve hits
            std::unordered_set<uint64_t> seen;
            for (int64_t i = 0; i < b.nrec; ++i) {
                const uint32_t* rr = &b.rec[static_cast<size_t>(i) * dr.wp.rec_words];
                seen.insert(static_cast<uint64_t>(rr[4]) | (static_cast<uint64_t>(rr[5]) << 32));
            }
            st.emitted = static_cast<int64_t>(seen.size());
            st.delta_evals = bp.cfg.count_visited ? st.delta_evals : -1;
            const int64_t free_bits = bp.d.kp1 - bp.d.p;
            st.delta_evals_computed = (st.iterations + st.walks) * free_bits;
            st.n_gpus = 1;
            *last = st;
        }
    } catch (const CudaFailure& e) {
        set_error(e.what());
        return LABS_ECUDA;
    }
    return LABS_OK;
}

void labs_bench_destroy(labs_bench_plan* plan) { delete plan; }

}  // extern "C"
