// engine.cpp -- host orchestration of the Step-1 GPU path and the C ABI
// (include/labs_gpu.h).  Replaces run_saw_pool (saw.cpp:218-267): the pool's walks are
// planned in the reference's order, cut into jobs that the per-device executors
// (runner.hpp) seed, walk and compact on the GPU, and the finished jobs are replayed on the
// host -- walk by walk, in the pool's order -- through DedupSink -> CountingSink semantics
// (candidate.hpp:84-99, saw.cpp:173-194) before reaching the caller's sink.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "host_util.hpp"
#include "runner.hpp"

namespace labs_b200 {

namespace {
thread_local std::string g_error;
}
void set_error(const std::string& msg) { g_error = msg; }

// Device contexts (streams, events, uploaded hash tables, grow-only job buffers) are kept
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
            n / 256, std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
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

constexpr int64_t kMaxBatchWalks = 1 << 20;  // walks per job (bounds the slot buffers)
constexpr int64_t kPipelineBatches = 16;     // independent pools: jobs per device (>= 2 waves each)
constexpr int64_t kQueueDepth = 3;           // jobs queued per device ahead of the replay
constexpr int64_t kPreseedMaxWalks = 1 << 22;  // independent pools up to this many walks are
                                               // seeded in one K3 launch (<= 512 MB of halves)
constexpr double kBatchTargetMs = 100.0;     // coupled pools: one batch runs about this long

// One run_saw_pool call.
//
// Independent pools (no quota / time / stop_at_energy, max_restarts > 0): every (walker,
// restart) walk depends only on (seed, walker, restart, prefixes[w mod P]) (SURVEY.md
// §8(e)), so the walkers are split over the devices by restriction class, each device runs
// its walker-major job list, and the replay merges the devices' walks back into the
// reference's --threads 1 order (walker, restart, iteration): the candidate list is
// identical to the reference's for any device count.
//
// Coupled pools (quota, stop_at_energy, time budget or unlimited restarts) couple the
// walkers through the stop flag (saw.cpp:153-170,204-208).  The pool is issued in batches
// of about kBatchTargetMs (sized from the measured walk rate, and from the remaining time
// budget), two in flight; the stop conditions are evaluated in delivery order between
// walks, exactly where the reference checks them, and a stop cancels the batches still
// running (at the deadline, the batches not yet being replayed).  With threads <= 1 the batches follow the --threads 1 order exactly (walker 0's
// restarts first; with unlimited restarts that is walker 0 alone, as in the reference).
// With threads > 1 every walker runs concurrently, as the reference's pool does when
// threads >= walkers (saw.cpp:242-257): each batch gives every unfinished walker its next
// restarts, round-robin, across all devices.
class Pool {
public:
    Pool(const labs_saw_config& cfg, const Derived& d, const WalkParams& wp, SinkChain& sink,
         PoolAccum& acc)
        : cfg_(cfg), d_(d), wp_(wp), sink_(sink), acc_(acc) {}

    ~Pool() { shutdown(true); }

    void run(int first, int ndev_use, int ngpu, const std::vector<uint32_t>& walkers,
             const std::chrono::steady_clock::time_point t0) {
        t0_ = t0;
        walkers_ = walkers;
        ngpu_ = ngpu;
        owner_.resize(walkers_.size());
        gen_.resize(walkers_.size());
        dev_walkers_.assign(static_cast<size_t>(ngpu), {});
        for (size_t i = 0; i < walkers_.size(); ++i) {
            const int g = static_cast<int>((walkers_[i] % static_cast<uint32_t>(d_.nprefix)) %
                                           static_cast<uint32_t>(ngpu));
            owner_[i] = g;
            gen_[i] = static_cast<uint32_t>(dev_walkers_[static_cast<size_t>(g)].size());
            dev_walkers_[static_cast<size_t>(g)].push_back(i);
        }
        for (int g = 0; g < ngpu; ++g) {
            runners_.push_back(acquire_runner(first + g % ndev_use, wp_));
            DeviceRunner& dr = *runners_.back();
            dr.seed = cfg_.seed;
            dr.d = &d_;
            dr.reserve_generators(dev_walkers_[static_cast<size_t>(g)].size());
        }
        for (auto& r : runners_) {
            ex_.emplace_back(new Executor(*r));
            ex_.back()->start();
        }
        if (timing_)
            std::fprintf(stderr, "[labs] pool t=%.2f ms: runners ready\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count());
        cur_.resize(static_cast<size_t>(ngpu));
        dev_kernel_ms_.assign(static_cast<size_t>(ngpu), 0.0);
        dev_seed_ms_.assign(static_cast<size_t>(ngpu), 0.0);
        const bool coupled = cfg_.candidate_quota > 0 || cfg_.stop_at_energy > 0 ||
                             cfg_.time_budget_s > 0 || cfg_.max_restarts == 0;
        if (coupled) run_coupled();
        else run_independent();
        for (int g = 0; g < ngpu; ++g) {  // device time = the slowest device
            acc_.st.kernel_ms = std::max(acc_.st.kernel_ms, dev_kernel_ms_[static_cast<size_t>(g)]);
            acc_.st.seed_ms = std::max(acc_.st.seed_ms, dev_seed_ms_[static_cast<size_t>(g)]);
        }
    }

    // Cancel whatever still runs, join the executors, return the runners to the pool
    // (only after a clean run: a failed device's state may be unusable).
    void shutdown(bool failed) {
        if (done_) return;
        done_ = true;
        for (auto& e : ex_) e->cancel();
        for (auto& e : ex_) e->stop();
        sink_.flush();  // before the jobs' record buffers are released
        cur_.clear();
        ex_.clear();
        if (!failed) release_runners(runners_);
        runners_.clear();
    }

private:
    const labs_saw_config& cfg_;
    const Derived& d_;
    WalkParams wp_;
    SinkChain& sink_;
    PoolAccum& acc_;
    std::chrono::steady_clock::time_point t0_;
    int ngpu_ = 1;
    bool done_ = false;
    std::vector<uint32_t> walkers_;
    std::vector<int> owner_;                        // per walker index: device
    std::vector<uint32_t> gen_;                     // per walker index: generator slot
    std::vector<std::vector<size_t>> dev_walkers_;  // per device: walker indices, in order
    std::vector<std::unique_ptr<DeviceRunner>> runners_;
    std::vector<std::unique_ptr<Executor>> ex_;
    struct Cursor {
        JobOut job;
        bool have = false;
        int64_t i = 0;
    };
    std::vector<Cursor> cur_;
    std::vector<double> dev_kernel_ms_, dev_seed_ms_;
    double ms_per_walk_ = 0;       // measured device time per walk at full residency
    double replay_ms_per_walk_ = 0;  // measured host replay time per walk (coupled pools)
    double wait_ms_ = 0;             // time the replay spent waiting for the devices
    double wall_ms_per_walk_ = 0;    // consume wall time per walk of the latest batch
    int64_t last_batch_ = 1;         // walks of the latest coupled batch
    const bool timing_ = std::getenv("LABS_TIMING") != nullptr;
    const bool shrink_ = !(std::getenv("LABS_TAIL_SHRINK") && std::string(std::getenv("LABS_TAIL_SHRINK")) == "0");
    // independent pools: per device, the next walk of its job list
    struct Gen {
        size_t k = 0;   // index into dev_walkers_[g]
        int64_t r = 0;
        int64_t off = 0;      // walks handed out so far (= offset into the preseeded halves)
        bool pre = false;     // the device's pool was preseeded
    };
    std::vector<Gen> feed_;
    std::vector<int64_t> chunk_;

    bool stopped() const { return sink_.stop || sink_.aborted || acc_.diverged != 0; }

    bool deadline_hit() const {
        return cfg_.time_budget_s > 0 &&
               std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count() >=
                   cfg_.time_budget_s;
    }

    Segment seg(size_t wi, int64_t r0, int64_t r1) const {
        Segment s;
        s.walker = walkers_[wi];
        s.r0 = r0;
        s.r1 = r1;
        s.gen = gen_[wi];
        return s;
    }

    // ---- independent pools
    void top_up() {
        if (feed_.empty()) return;
        const int64_t R = cfg_.max_restarts;
        for (int g = 0; g < ngpu_; ++g) {
            Executor& e = *ex_[static_cast<size_t>(g)];
            Gen& f = feed_[static_cast<size_t>(g)];
            const auto& wl = dev_walkers_[static_cast<size_t>(g)];
            const int64_t total = static_cast<int64_t>(wl.size()) * R;
            const int64_t half_wave = std::max<int64_t>(1, runners_[static_cast<size_t>(g)]->resident / 2);
            while (e.pushed() - e.popped() < kQueueDepth && f.k < wl.size()) {
                Job job;
                if (f.pre) job.pool_off = f.off;
                // the last jobs shrink (half the remainder, down to half a wave): the host replay
                // of the final job is all that follows the last kernel
                const int64_t left = total - f.off;
                const int64_t chunk = std::min(chunk_[static_cast<size_t>(g)],
                                               shrink_ && left <= 2 * chunk_[static_cast<size_t>(g)]
                                                   ? std::max(half_wave, (left + 1) / 2) : left);
                while (job.nwalks < chunk && f.k < wl.size()) {
                    const int64_t take = std::min(R - f.r, chunk - job.nwalks);
                    job.segs.push_back(seg(wl[f.k], f.r, f.r + take));
                    job.nwalks += take;
                    f.r += take;
                    if (f.r == R) {
                        ++f.k;
                        f.r = 0;
                    }
                }
                f.off += job.nwalks;
                e.push(std::move(job));
            }
        }
    }

    void run_independent() {
        const int64_t R = cfg_.max_restarts;
        const char* nb_env = std::getenv("LABS_PIPELINE_BATCHES");  // (A/B knob)
        const int64_t nb = std::max<int64_t>(1, nb_env ? std::atoll(nb_env) : kPipelineBatches);
        feed_.assign(static_cast<size_t>(ngpu_), Gen{});
        chunk_.assign(static_cast<size_t>(ngpu_), 1);
        for (int g = 0; g < ngpu_; ++g) {
            const int64_t total = static_cast<int64_t>(dev_walkers_[static_cast<size_t>(g)].size()) * R;
            const int64_t resident = runners_[static_cast<size_t>(g)]->resident;
            chunk_[static_cast<size_t>(g)] = std::max<int64_t>(1, std::min<int64_t>(
                kMaxBatchWalks, nb == 1 ? total : std::max<int64_t>(2 * resident, (total + nb - 1) / nb)));
        }
        // one K3 launch seeds each device's whole pool before the first job (a per-job K3
        // would wait at every job boundary for the other slot's walk blocks to free an SM)
        const char* pre_env = std::getenv("LABS_PRESEED");  // (A/B, tests: 0 = K3 per job)
        const bool preseed = !(pre_env && std::string(pre_env) == "0");
        for (int g = 0; g < ngpu_ && preseed; ++g) {
            const auto& wl = dev_walkers_[static_cast<size_t>(g)];
            const int64_t total = static_cast<int64_t>(wl.size()) * R;
            if (total <= 0 || total > kPreseedMaxWalks) continue;
            std::vector<Segment> segs;
            segs.reserve(wl.size());
            for (size_t wi : wl) segs.push_back(seg(wi, 0, R));
            runners_[static_cast<size_t>(g)]->preseed(segs, total);
            feed_[static_cast<size_t>(g)].pre = true;
        }
        top_up();
        for (size_t wi = 0; wi < walkers_.size() && !stopped(); ++wi)
            for (int64_t r = 0; r < R && !stopped(); ++r) deliver_next(wi, r);
    }

    // ---- coupled pools
    void run_coupled() {
        const bool exact = cfg_.threads <= 1;
        const int64_t lim = cfg_.max_restarts > 0 ? cfg_.max_restarts : INT64_MAX;
        std::vector<int64_t> next_r(walkers_.size(), 0);
        size_t ex_wi = 0, cyc = 0;
        int64_t ex_r = 0;
        int64_t resident_all = 0;
        for (auto& r : runners_) resident_all += r->resident;
        std::deque<std::vector<size_t>> issued;  // per batch: walker index of each segment
        std::deque<std::vector<Segment>> issued_segs;
        bool exhausted = false;
        const auto make_batch = [&](int64_t n, std::vector<size_t>& idx, std::vector<Segment>& segs) {
            int64_t nw = 0;
            if (exact) {
                while (nw < n && ex_wi < walkers_.size()) {
                    const int64_t take = std::min(lim - ex_r, n - nw);
                    idx.push_back(ex_wi);
                    segs.push_back(seg(ex_wi, ex_r, ex_r + take));
                    nw += take;
                    ex_r += take;
                    if (ex_r >= lim) {
                        ++ex_wi;
                        ex_r = 0;
                    }
                }
                return nw;
            }
            int64_t active = 0;
            for (size_t i = 0; i < walkers_.size(); ++i) active += next_r[i] < lim ? 1 : 0;
            if (active == 0) return int64_t(0);
            const int64_t c = std::max<int64_t>(1, n / active);
            for (size_t step = 0; step < walkers_.size() && nw < n; ++step) {
                const size_t i = (cyc + step) % walkers_.size();
                if (next_r[i] >= lim) continue;
                const int64_t take = std::min({c, lim - next_r[i], n - nw});
                idx.push_back(i);
                segs.push_back(seg(i, next_r[i], next_r[i] + take));
                next_r[i] += take;
                nw += take;
                if (nw >= n) cyc = (i + 1) % walkers_.size();
            }
            return nw;
        };
        // (the first batch is issued even when device setup used up a tiny budget: the
        // reference's walkers all start their first walk at once)
        bool first_batch = true;
        const auto issue = [&]() {
            if (exhausted || stopped() || (deadline_hit() && !first_batch)) return false;
            first_batch = false;
            double target = kBatchTargetMs;
            if (cfg_.time_budget_s > 0) {
                const double left = cfg_.time_budget_s * 1e3 -
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
                target = std::min(target, std::max(1.0, left / 3));
            }
            // The pipeline runs at the slower of the devices and the host replay (a loose
            // threshold makes the replay -- dedup of every hit -- the bound).  The first
            // batches are small (one walk per walker, at most one wave) so that the rates are
            // measured before the batches grow (at most 4x per batch) to ~target ms.
            int64_t n = std::min<int64_t>(resident_all, static_cast<int64_t>(walkers_.size()));
            if (ms_per_walk_ > 0) {
                n = std::max<int64_t>(resident_all, static_cast<int64_t>(ngpu_ * target / ms_per_walk_));
                if (replay_ms_per_walk_ > 0)
                    n = std::min<int64_t>(n, static_cast<int64_t>(target / replay_ms_per_walk_));
                // the whole pipeline's pace (device, job post-processing, replay) per walk
                if (wall_ms_per_walk_ > 0)
                    n = std::min<int64_t>(n, static_cast<int64_t>(target / wall_ms_per_walk_));
                n = std::max<int64_t>(1, std::min<int64_t>(n, 4 * last_batch_));
            }
            n = std::min<int64_t>(n, kMaxBatchWalks * ngpu_);
            std::vector<size_t> idx;
            std::vector<Segment> segs;
            last_batch_ = make_batch(n, idx, segs);
            if (last_batch_ == 0) {
                exhausted = true;
                return false;
            }
            std::vector<Job> jobs(static_cast<size_t>(ngpu_));
            for (size_t j = 0; j < segs.size(); ++j) {
                Job& job = jobs[static_cast<size_t>(owner_[idx[j]])];
                job.segs.push_back(segs[j]);
                job.nwalks += segs[j].r1 - segs[j].r0;
            }
            for (int g = 0; g < ngpu_; ++g)
                if (jobs[static_cast<size_t>(g)].nwalks > 0)
                    ex_[static_cast<size_t>(g)]->push(std::move(jobs[static_cast<size_t>(g)]));
            if (timing_)
                std::fprintf(stderr, "[labs] t=%.1f ms issue batch of %lld walks (%zu segs; device %.4f, "
                             "replay %.4f, wall %.4f ms/walk)\n",
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count(),
                             static_cast<long long>(last_batch_), segs.size(), ms_per_walk_, replay_ms_per_walk_,
                             wall_ms_per_walk_);
            issued.push_back(std::move(idx));
            issued_segs.push_back(std::move(segs));
            return true;
        };
        while (issued.size() < 2 && issue()) {
        }
        bool consumed_any = false;
        while (!issued.empty() && !stopped()) {
            // at the deadline the batches whose replay has not begun are dropped (cancelled on
            // the device): the reference starts no walk after its deadline (saw.cpp:204-208),
            // and the overshoot stays one batch of replay
            if (consumed_any && deadline_hit()) break;
            consumed_any = true;
            const std::vector<size_t> idx = std::move(issued.front());
            const std::vector<Segment> segs = std::move(issued_segs.front());
            issued.pop_front();
            issued_segs.pop_front();
            const auto ta = std::chrono::steady_clock::now();
            const double wait0 = wait_ms_;
            int64_t nw = 0;
            for (size_t j = 0; j < segs.size() && !stopped(); ++j)
                for (int64_t r = segs[j].r0; r < segs[j].r1 && !stopped(); ++r, ++nw)
                    deliver_next(idx[j], r);
            // host replay time per walk (the waits for the devices excluded), and the batch's
            // wall time per walk (waits included)
            if (nw > 0) {
                const double wall = std::chrono::duration<double, std::milli>(
                    std::chrono::steady_clock::now() - ta).count();
                replay_ms_per_walk_ = std::max(0.0, wall - (wait_ms_ - wait0)) / static_cast<double>(nw);
                wall_ms_per_walk_ = wall / static_cast<double>(nw);
            }
            while (issued.size() < 2 && issue()) {
            }
        }
    }

    // ---- replay: the next walk of walker index wi (restart r) from its device's jobs
    void deliver_next(size_t wi, int64_t r) {
        const int g = owner_[wi];
        Cursor& c = cur_[static_cast<size_t>(g)];
        while (!c.have || c.i >= static_cast<int64_t>(c.job.walk_walker.size())) {
            if (c.have) {
                // the job is replayed: hand its candidates to the sink now, while the
                // devices still run (only the last job's flush is left after the last kernel)
                sink_.flush();
                c.have = false;
            }
            top_up();
            const auto tw = std::chrono::steady_clock::now();
            c.job = ex_[static_cast<size_t>(g)]->pop();
            wait_ms_ += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw).count();
            c.have = true;
            c.i = 0;
            account(g, c.job);
        }
        const int64_t i = c.i++;
        const JobOut& b = c.job;
        if (b.walk_walker[static_cast<size_t>(i)] != walkers_[wi] ||
            b.walk_restart[static_cast<size_t>(i)] != r)
            throw CudaFailure("walk replay out of order");
        const int64_t* s = &b.stats[static_cast<size_t>(i) * kWalkStatWords];
        for (int64_t v = b.start[static_cast<size_t>(i)]; v < b.start[static_cast<size_t>(i) + 1]; ++v)
            sink_.deliver(walkers_[wi], r, b.views[static_cast<size_t>(v)]);
        ++acc_.st.walks;
        acc_.st.iterations += s[kWsIterations];
        acc_.st.emitted_raw += s[kWsEmitted];
        acc_.st.delta_evals += s[kWsDeltaEvals] >= 0 ? s[kWsDeltaEvals] : 0;
        acc_.st.exhausted_walks += s[kWsExhausted];
        acc_.st.wide_iterations += s[kWsWideIters];
        acc_.diverged += s[kWsDiverged];
        // offer_best (saw.cpp:160-169)
        if (!acc_.best_set || s[kWsBest] < acc_.st.best_energy) {
            acc_.st.best_energy = s[kWsBest];
            acc_.best_set = true;
            if (cfg_.stop_at_energy > 0 && s[kWsBest] <= cfg_.stop_at_energy) sink_.stop = true;
        }
    }

    void account(int g, const JobOut& b) {
        dev_kernel_ms_[static_cast<size_t>(g)] += b.kernel_ms;
        dev_seed_ms_[static_cast<size_t>(g)] += b.seed_ms;
        acc_.st.h2d_bytes += b.h2d;
        acc_.st.d2h_bytes += b.d2h;
        const int64_t nw = static_cast<int64_t>(b.walk_walker.size());
        const int64_t res = runners_[static_cast<size_t>(g)]->resident;
        if (nw > 0 && b.kernel_ms > 0)
            ms_per_walk_ = b.kernel_ms / static_cast<double>(std::max(nw, res));
    }
};

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
    if (first >= ndev_avail) {
        set_error("device ordinal out of range");
        return LABS_ENODEV;
    }
    // n_gpus class shards run concurrently, shard g on device first + g (mod the devices
    // available from `first`); more shards than devices share a device (separate streams)
    const int ngpu = std::max(1, cfg.n_gpus);
    const int ndev_use = std::max(1, ndev_avail - first);
    const int sidx = cfg.shard_count > 1 ? cfg.shard_index : 0;
    const int scnt = cfg.shard_count > 1 ? cfg.shard_count : 1;
    std::vector<uint32_t> walkers = walker_list(cfg, d, sidx, scnt);
    if (cfg.max_restarts < 0) walkers.clear();  // (saw.cpp:202: no restart runs)

    PoolAccum acc;
    SinkChain sink{};
    sink.cfg = &cfg;
    sink.d = &d;
    sink.emit = emit;
    sink.emit_batch = emit_batch;
    sink.user = user;
    const bool timing = std::getenv("LABS_TIMING") != nullptr;
    const auto mark = [&](const char* what) {
        if (timing)
            std::fprintf(stderr, "[labs] pool t=%.2f ms: %s\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
                         what);
    };
    mark("configured");
    if (!walkers.empty()) {
        Pool pool(cfg, d, wp, sink, acc);
        try {
            pool.run(first, ndev_use, ngpu, walkers, t0);
            mark("replayed");
            pool.shutdown(false);
            mark("shut down");
        } catch (const CudaFailure& e) {
            pool.shutdown(true);
            set_error(e.what());
            return LABS_ECUDA;
        } catch (const std::bad_alloc&) {
            pool.shutdown(true);
            set_error("out of host memory");
            return LABS_ECUDA;
        }
    }
    if (acc.diverged) {
        set_error("saw walk energy bookkeeping diverged");
        return LABS_ELOGIC;
    }
    sink.flush();
    mark("flushed");
    acc.st.emitted = sink.emitted;
    acc.st.best_energy = acc.best_set ? acc.st.best_energy : 0;
    acc.st.delta_evals = cfg.count_visited ? acc.st.delta_evals : -1;
    int64_t free_bits = d.kp1 - d.p;
    acc.st.delta_evals_computed = (acc.st.iterations + acc.st.walks) * (free_bits > 0 ? free_bits : 0);
    acc.st.n_gpus = ngpu;
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
        std::unique_ptr<DeviceRunner> dr = acquire_runner(0, wp);
        std::vector<uint32_t> hb(static_cast<size_t>(nwalks) * wp.hw, 0u);
        for (int64_t w = 0; w < nwalks; ++w)
            for (int i = 0; i < kp1; ++i)
                if (halves[w * kp1 + i] > 0) hb[static_cast<size_t>(w) * wp.hw + (i >> 5)] |= 1u << (i & 31);
        DevBuf<int> dscore, dcorr;
        if (deltas_out) {
            dscore.reserve(static_cast<size_t>(nwalks) * kp1);
            dcorr.reserve(static_cast<size_t>(nwalks) * std::max(1, kp1 - 1));
        }
        Job job;
        job.nwalks = nwalks;
        job.host_halves = hb.data();
        job.score_out = deltas_out ? dscore.p : nullptr;
        job.corr_out = deltas_out ? dcorr.p : nullptr;
        JobOut b = dr->run_sync(job);
        if (deltas_out) {
            std::vector<int> hs(static_cast<size_t>(nwalks) * kp1), hc(static_cast<size_t>(nwalks) * (kp1 - 1));
            LABS_CUDA(cudaMemcpy(hs.data(), dscore.p, hs.size() * 4, cudaMemcpyDeviceToHost));
            if (!hc.empty())
                LABS_CUDA(cudaMemcpy(hc.data(), dcorr.p, hc.size() * 4, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < hs.size(); ++i) deltas_out[i] = hs[i];
            if (corr_out)
                for (size_t i = 0; i < hc.size(); ++i) corr_out[i] = hc[i];
        }
        std::vector<std::unique_ptr<DeviceRunner>> keep;
        keep.push_back(std::move(dr));
        release_runners(keep);
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
                for (int64_t v = b.start[static_cast<size_t>(w)]; v < b.start[static_cast<size_t>(w) + 1]; ++v) {
                    const WalkRecordView& rv = b.views[static_cast<size_t>(v)];
                    half_bits_to_signs(rv.half, kp1, half.data());
                    if (on_rec(user, w, rv.iteration, rv.energy, half.data(), kp1) != 0) return LABS_EABORT;
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
    out->kernel = err.empty() ? wp.kernel : 0;
    out->lanes_per_walk = err.empty() ? wp.lpw : 0;
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

int labs_saw_prepare(const labs_saw_config* cfg) {
    if (!cfg) {
        set_error("null config");
        return LABS_EINVAL;
    }
    Derived d;
    std::string err = derive(*cfg, d);
    WalkParams wp;
    if (err.empty()) err = walk_params_for(d, cfg->count_visited != 0, cfg->debug_check_energy != 0, wp);
    if (!err.empty()) {
        set_error(err);
        return LABS_EINVAL;
    }
    const int ndev_avail = device_count();
    const int first = std::max(0, cfg->device);
    if (ndev_avail <= 0 || first >= ndev_avail) {
        set_error("no CUDA device available (the Step-1 engine has no CPU fallback)");
        return LABS_ENODEV;
    }
    const int ndev_use = std::max(1, ndev_avail - first);
    std::vector<std::unique_ptr<DeviceRunner>> rs;
    try {
        for (int g = 0; g < std::max(1, cfg->n_gpus); ++g) rs.push_back(acquire_runner(first + g % ndev_use, wp));
    } catch (const CudaFailure& e) {
        set_error(e.what());
        return LABS_ECUDA;
    }
    release_runners(rs);  // (the next pool with this geometry takes them from the pool)
    return LABS_OK;
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
        for (uint32_t w : walker_list(bp.cfg, bp.d, sidx, scnt)) {
            Segment g;
            g.walker = w;
            g.r0 = 0;
            g.r1 = cfg->max_restarts;
            g.gen = static_cast<uint32_t>(bp.segs.size());
            bp.segs.push_back(g);
        }
        bp.nwalks = static_cast<int64_t>(bp.segs.size()) * cfg->max_restarts;
        if (bp.nwalks > kMaxBatchWalks) throw CudaFailure("bench plan larger than one batch");
        bp.dr->seed = bp.cfg.seed;
        bp.dr->d = &bp.d;
        bp.dr->reserve_generators(bp.segs.size());
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
        JobOut b;
        bp.l2_scratch.reserve(BenchPlan::kL2Flush);
        Job job;
        job.segs = bp.segs;
        job.nwalks = bp.nwalks;
        for (int r = 0; r < reps; ++r) {
            LABS_CUDA(cudaMemsetAsync(bp.l2_scratch.p, r & 0xff, BenchPlan::kL2Flush, 0));
            LABS_CUDA(cudaDeviceSynchronize());
            b = dr.run_sync(job);
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
            for (const WalkRecordView& v : b.views) seen.insert(v.hash);
            st.emitted = static_cast<int64_t>(seen.size());
            st.delta_evals = bp.cfg.count_visited ? st.delta_evals : -1;
            const int64_t free_bits = bp.d.kp1 - bp.d.p;
            st.delta_evals_computed = (st.iterations + st.walks) * free_bits;
            st.h2d_bytes = b.h2d;
            st.d2h_bytes = b.d2h;
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
