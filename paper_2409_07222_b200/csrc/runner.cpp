// runner.cpp -- per-device execution of Step-1 walk jobs (see runner.hpp).
#include "runner.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>

namespace labs_b200 {

cudaError_t launch_saw_walk(const WalkParams& P, int grid, cudaStream_t st, int* score_out,
                            int* corr_out);
cudaError_t launch_saw_seed(const SeedParams& P, cudaStream_t st);
cudaError_t preload_saw_seed();
int walk_blocks_per_sm(WalkParams& P);  // (also places the fm table)
size_t walk_smem_bytes(const WalkParams& P);

namespace {
constexpr int64_t kDefaultRingSlots = 1 << 16;

int64_t ring_slots_from_env() {
    // LABS_RING_SLOTS (tests): a small ring forces drains while the launch runs
    const char* e = std::getenv("LABS_RING_SLOTS");
    int64_t n = e ? std::atoll(e) : kDefaultRingSlots;
    int64_t p2 = 16;
    while (p2 < n && p2 < (int64_t(1) << 24)) p2 <<= 1;
    return p2;
}
}  // namespace

void JobOut::group(int rec_words) {
    const int64_t nw = static_cast<int64_t>(walk_walker.size());
    views.resize(static_cast<size_t>(nrec));
    start.assign(static_cast<size_t>(nw) + 1, 0);
    for (int64_t i = 0; i < nrec; ++i) {
        const uint32_t* r = &rec[static_cast<size_t>(i) * rec_words];
        views[static_cast<size_t>(i)] = WalkRecordView{
            static_cast<int64_t>(r[0]), static_cast<int64_t>(r[1]),
            static_cast<int64_t>(static_cast<int32_t>(r[2])),
            static_cast<uint64_t>(r[4]) | (static_cast<uint64_t>(r[5]) << 32), r + kRecHeader};
        ++start[static_cast<size_t>(r[0]) + 1];
    }
    std::sort(views.begin(), views.end(), [](const WalkRecordView& a, const WalkRecordView& c) {
        return a.walk != c.walk ? a.walk < c.walk : a.iteration < c.iteration;
    });
    for (int64_t w = 0; w < nw; ++w) start[static_cast<size_t>(w) + 1] += start[static_cast<size_t>(w)];
}

// ------------------------------------------------------------------ DeviceRunner
DeviceRunner::~DeviceRunner() {
    if (!drain_st_) return;
    cudaSetDevice(dev);
    for (Slot& S : slot_) {
        if (S.st) cudaStreamSynchronize(S.st);
        for (cudaEvent_t e : {S.ev_s0, S.ev_s1, S.ev_k0, S.ev_k1, S.ev_done})
            if (e) cudaEventDestroy(e);
        if (S.st) cudaStreamDestroy(S.st);
    }
    for (cudaEvent_t e : {pre_ev0_, preseed_ev_})
        if (e) cudaEventDestroy(e);
    cudaStreamDestroy(drain_st_);
}

void DeviceRunner::init(int device, const WalkParams& params) {
    dev = device;
    wp = params;
    LABS_CUDA(cudaSetDevice(dev));
    LABS_CUDA(cudaStreamCreateWithFlags(&drain_st_, cudaStreamNonBlocking));
    for (Slot& S : slot_) {
        LABS_CUDA(cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&S.ev_s0, &S.ev_s1, &S.ev_k0, &S.ev_k1, &S.ev_done})
            LABS_CUDA(cudaEventCreate(e));
    }
    LABS_CUDA(cudaEventCreate(&pre_ev0_));
    LABS_CUDA(cudaEventCreate(&preseed_ev_));
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
    LABS_CUDA(cudaMemcpy(fm.p, hfm.data(), hfm.size() * 8, cudaMemcpyHostToDevice));
    LABS_CUDA(cudaMemcpy(tab.p, htab.data(), htab.size() * 8, cudaMemcpyHostToDevice));
    LABS_CUDA(cudaMemcpy(tabfull.p, hfull.data(), hfull.size() * 8, cudaMemcpyHostToDevice));
    wp.fm = fm.p;
    wp.tab = tab.p;
    wp.tabfull = tabfull.p;
    wp.salt0 = tt.salt[0][kp1];
    wp.salt1 = tt.salt[1][kp1];
    wp.salt_full = tt.salt[0][L];
    int sms = 0;
    LABS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int bps = std::max(1, walk_blocks_per_sm(wp));  // (loads the walk kernel's module)
    LABS_CUDA(preload_saw_seed());
    grid_cap = sms * bps;
    resident = static_cast<int64_t>(grid_cap) * wp.walks_per_block;
    if (std::getenv("LABS_TIMING"))
        std::fprintf(stderr, "[labs] dev %d: kernel %d, L=%d, lanes/walk %d, R %d, %d blocks/SM of %d walks, "
                     "%d B shared per block, resident %lld walks\n", dev, wp.kernel, wp.L, wp.lpw, wp.R, bps,
                     wp.walks_per_block, static_cast<int>(walk_smem_bytes(wp)),
                     static_cast<long long>(resident));
    ring_slots = ring_slots_from_env();
    for (Slot& S : slot_) {
        S.ctr.reserve(4);
        S.ring.reserve(static_cast<size_t>(ring_slots) * wp.rec_words);
        S.tag.reserve(static_cast<size_t>(ring_slots));
        S.h_ring.reserve(static_cast<size_t>(ring_slots) * wp.rec_words);
        S.h_tag.reserve(static_cast<size_t>(ring_slots));
        LABS_CUDA(cudaMemset(S.tag.p, 0, static_cast<size_t>(ring_slots) * 4));
        S.h_ctr.reserve(4);
        S.h_head.reserve(1);
        S.h_tail.reserve(1);
        S.h_cancel.reserve(1);
    }
}

// Allocations (cudaFree, cudaFreeHost) synchronise the device: a slot may only grow while
// the other slot is idle, or a launch waiting for its ring to drain would deadlock the
// thread that drains it.  The executor checks fits() and lets the other slot finish first.
bool DeviceRunner::fits(int s, const Job& job) const {
    const Slot& S = slot_[s];
    const size_t nw = static_cast<size_t>(std::max<int64_t>(job.nwalks, 1));
    const size_t nseg = job.segs.size();
    if (ring_slots_from_env() != ring_slots) return false;
    if (nw * kWalkStatWords > S.stats.n || nw * kWalkStatWords > S.h_stats.n) return false;
    if (job.pool_off >= 0) return true;  // (halves from the pool buffer)
    if (nw * wp.hw > S.halves.n) return false;
    if (job.host_halves && nw * wp.hw > S.h_halves.n) return false;
    if (!job.host_halves && nseg > 0 && !S.sb.fits(nseg)) return false;
    return true;
}

void DeviceRunner::launch(int s, const Job& job) {
    Slot& S = slot_[s];
    if (S.busy) throw CudaFailure("runner slot busy");
    const int64_t nw = job.nwalks;
    const int nseg = static_cast<int>(job.segs.size());
    S.out = JobOut();
    S.out.walk_walker.reserve(static_cast<size_t>(nw));
    S.out.walk_restart.reserve(static_cast<size_t>(nw));
    for (const Segment& g : job.segs)
        for (int64_t r = g.r0; r < g.r1; ++r) {
            S.out.walk_walker.push_back(g.walker);
            S.out.walk_restart.push_back(r);
        }
    if (job.host_halves) {  // seed-table mode: walks are numbered 0..nw-1 only
        S.out.walk_walker.assign(static_cast<size_t>(nw), 0u);
        S.out.walk_restart.assign(static_cast<size_t>(nw), 0);
    }
    if (static_cast<int64_t>(S.out.walk_walker.size()) != nw)
        throw CudaFailure("job walk count mismatch");
    // (growth happens only while the other slot is idle -- see fits() -- so both slots are
    // sized for the job: the next one then launches without waiting)
    for (Slot& T : slot_) {
        if (&T != &S && T.busy) continue;
        T.stats.reserve(static_cast<size_t>(std::max<int64_t>(nw, 1)) * kWalkStatWords);
        T.h_stats.reserve(static_cast<size_t>(std::max<int64_t>(nw, 1)) * kWalkStatWords);
        if (job.pool_off >= 0) continue;
        T.halves.reserve(static_cast<size_t>(std::max<int64_t>(nw, 1)) * wp.hw);
        if (!job.host_halves && nseg > 0) T.sb.reserve(static_cast<size_t>(nseg));
    }
    S.seeded = false;
    const int64_t want_slots = ring_slots_from_env();  // (tests shrink it per call)
    if (want_slots != ring_slots) {
        ring_slots = want_slots;
        for (Slot& T : slot_) {
            if (T.busy) throw CudaFailure("ring resize while a launch runs");
            T.ring.reserve(static_cast<size_t>(ring_slots) * wp.rec_words);
            T.tag.reserve(static_cast<size_t>(ring_slots));
            T.h_ring.reserve(static_cast<size_t>(ring_slots) * wp.rec_words);
            T.h_tag.reserve(static_cast<size_t>(ring_slots));
            LABS_CUDA(cudaMemset(T.tag.p, 0, static_cast<size_t>(ring_slots) * 4));
            T.seq0 = 0;
        }
    }
    if (job.host_halves) {
        const size_t words = static_cast<size_t>(nw) * wp.hw;
        S.h_halves.reserve(words);
        std::memcpy(S.h_halves.p, job.host_halves, words * 4);
        LABS_CUDA(cudaMemcpyAsync(S.halves.p, S.h_halves.p, words * 4, cudaMemcpyHostToDevice, S.st));
        S.out.h2d += static_cast<int64_t>(words) * 4;
    } else if (job.pool_off >= 0) {
        if (job.pool_off + nw > pool_walks_) throw CudaFailure("job outside the preseeded pool");
        LABS_CUDA(cudaStreamWaitEvent(S.st, preseed_ev_, 0));
        S.out.h2d += pending_h2d_;
        pending_h2d_ = 0;
        if (!preseed_timed_) {  // (the preseed's K3 time is reported with the first job)
            S.seeded = true;
            S.seed_from = pre_ev0_;
            S.seed_to = preseed_ev_;
            preseed_timed_ = true;
        }
    } else if (nseg > 0) {
        S.out.h2d += seed_into(S.st, S.sb, job.segs, S.halves.p, S.ev_s0, S.ev_s1);
        S.seeded = true;
        S.seed_from = S.ev_s0;
        S.seed_to = S.ev_s1;
    }
    LABS_CUDA(cudaMemsetAsync(S.ctr.p, 0, 4 * sizeof(unsigned long long), S.st));
    WalkParams P = wp;
    P.nwalks = nw;
    P.halves = job.pool_off >= 0 ? pool_halves.p + job.pool_off * wp.hw : S.halves.p;
    P.rec = S.ring.p;
    P.rec_tag = S.tag.p;
    P.rec_seq0 = S.seq0;
    P.rec_cap = ring_slots;
    P.rec_count = S.ctr.p;
    P.walk_next = S.ctr.p + 1;
    P.rec_tail = S.ctr.p + 2;
    P.ctl = reinterpret_cast<int*>(S.ctr.p + 3);
    P.walk_stats = S.stats.p;
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(grid_cap, (nw + P.walks_per_block - 1) / P.walks_per_block)));
    LABS_CUDA(cudaEventRecord(S.ev_k0, S.st));
    if (nw > 0) LABS_CUDA(launch_saw_walk(P, grid, S.st, job.score_out, job.corr_out));
    LABS_CUDA(cudaEventRecord(S.ev_k1, S.st));
    LABS_CUDA(cudaMemcpyAsync(S.h_ctr.p, S.ctr.p, 4 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, S.st));
    if (nw > 0) {
        LABS_CUDA(cudaMemcpyAsync(S.h_stats.p, S.stats.p,
                                  static_cast<size_t>(nw) * kWalkStatWords * 8,
                                  cudaMemcpyDeviceToHost, S.st));
    }
    LABS_CUDA(cudaEventRecord(S.ev_done, S.st));
    S.nwalks = nw;
    S.tail = 0;
    S.cancel_sent = false;
    S.busy = true;
}

int64_t DeviceRunner::seed_into(cudaStream_t st, SeedBufs& B, const std::vector<Segment>& segs,
                                uint32_t* halves, cudaEvent_t ev0, cudaEvent_t ev1) {
    const int nseg = static_cast<int>(segs.size());
    int64_t off = 0;
    for (int i = 0; i < nseg; ++i) {
        const Segment& g = segs[static_cast<size_t>(i)];
        B.h_seg32.p[i] = g.walker;
        B.h_seg32.p[nseg + i] = d->prefix_bits[g.walker % static_cast<uint32_t>(d->nprefix)];
        B.h_seg32.p[2 * nseg + i] = g.gen;
        B.h_seg64.p[i] = g.r1 - g.r0;
        B.h_seg64.p[nseg + i] = off;
        B.h_init.p[i] = g.r0 == 0 ? 1 : 0;
        off += g.r1 - g.r0;
    }
    LABS_CUDA(cudaMemcpyAsync(B.seg32.p, B.h_seg32.p, 12 * static_cast<size_t>(nseg),
                              cudaMemcpyHostToDevice, st));
    LABS_CUDA(cudaMemcpyAsync(B.seg64.p, B.h_seg64.p, 16 * static_cast<size_t>(nseg),
                              cudaMemcpyHostToDevice, st));
    LABS_CUDA(cudaMemcpyAsync(B.seg_init.p, B.h_init.p, 4 * static_cast<size_t>(nseg),
                              cudaMemcpyHostToDevice, st));
    SeedParams sp{};
    sp.kp1 = wp.kp1;
    sp.p = wp.p;
    sp.hw = wp.hw;
    sp.nseg = nseg;
    sp.seed = seed;
    sp.walker_ids = B.seg32.p;
    sp.prefix_bits = B.seg32.p + nseg;
    sp.seg_slot = B.seg32.p + 2 * nseg;
    sp.seg_restarts = B.seg64.p;
    sp.seg_offset = B.seg64.p + nseg;
    sp.seg_init = B.seg_init.p;
    sp.rng_state = rng.p;
    sp.halves = halves;
    // generator streams continue across jobs: K3 launches run in job order
    if (last_seed_) LABS_CUDA(cudaStreamWaitEvent(st, last_seed_, 0));
    LABS_CUDA(cudaEventRecord(ev0, st));
    LABS_CUDA(launch_saw_seed(sp, st));
    LABS_CUDA(cudaEventRecord(ev1, st));
    last_seed_ = ev1;
    return 32 * static_cast<int64_t>(nseg);
}

void DeviceRunner::preseed(const std::vector<Segment>& segs, int64_t nwalks) {
    for (const Slot& S : slot_)
        if (S.busy) throw CudaFailure("preseed on a busy runner");
    pool_halves.reserve(static_cast<size_t>(std::max<int64_t>(nwalks, 1)) * wp.hw);
    pool_sb.reserve(std::max<size_t>(segs.size(), 1));
    pending_h2d_ += seed_into(slot_[0].st, pool_sb, segs, pool_halves.p, pre_ev0_, preseed_ev_);
    pool_walks_ = nwalks;
    preseed_timed_ = false;
}

bool DeviceRunner::done(int s) {
    const cudaError_t e = cudaEventQuery(slot_[s].ev_done);
    if (e == cudaErrorNotReady) return false;
    LABS_CUDA(e);
    return true;
}

void DeviceRunner::cancel(int s) {
    Slot& S = slot_[s];
    if (!S.busy || S.cancel_sent) return;
    *S.h_cancel.p = 1;
    LABS_CUDA(cudaMemcpyAsync(reinterpret_cast<int*>(S.ctr.p + 3) + 1, S.h_cancel.p, sizeof(int),
                              cudaMemcpyHostToDevice, drain_st_));
    LABS_CUDA(cudaStreamSynchronize(drain_st_));
    S.cancel_sent = true;
    S.out.cancelled = true;
}

// Copy ring slots [S.tail, head) to the job's record list.  While the launch runs (final =
// false) only slots whose tag is already published are taken (tags first, then the records:
// a tag is written after its record's fence), and the new tail is written back so that
// warps waiting for space continue.  After the launch every reserved slot is complete.
void DeviceRunner::drain(Slot& S, unsigned long long head, bool final) {
    const int rw = wp.rec_words;
    const unsigned long long cap = static_cast<unsigned long long>(ring_slots);
    cudaStream_t st = final ? S.st : drain_st_;
    unsigned long long n = head - S.tail;
    if (n == 0) return;
    if (n > cap) n = cap;  // (cannot happen: writers wait for the tail)
    const auto ranges = [&](unsigned long long from, unsigned long long count,
                            auto&& fn) {  // [from, from+count) split at the ring's end
        const unsigned long long a = from & (cap - 1);
        const unsigned long long first = std::min(count, cap - a);
        fn(a, first, 0ull);
        if (first < count) fn(0ull, count - first, first);
    };
    unsigned long long ready = n;
    if (!final) {
        ranges(S.tail, n, [&](unsigned long long a, unsigned long long c, unsigned long long o) {
            LABS_CUDA(cudaMemcpyAsync(S.h_tag.p + o, S.tag.p + a, c * 4, cudaMemcpyDeviceToHost, st));
        });
        LABS_CUDA(cudaStreamSynchronize(st));
        S.out.d2h += static_cast<int64_t>(n) * 4;
        ready = 0;
        while (ready < n && S.h_tag.p[ready] == static_cast<uint32_t>(S.seq0 + S.tail + ready + 1)) ++ready;
        if (ready == 0) return;
    }
    ranges(S.tail, ready, [&](unsigned long long a, unsigned long long c, unsigned long long o) {
        LABS_CUDA(cudaMemcpyAsync(S.h_ring.p + o * rw, S.ring.p + a * rw, c * rw * 4,
                                  cudaMemcpyDeviceToHost, st));
    });
    LABS_CUDA(cudaStreamSynchronize(st));
    const size_t old = S.out.rec.size();
    S.out.rec.resize(old + static_cast<size_t>(ready) * rw);
    std::memcpy(S.out.rec.data() + old, S.h_ring.p, static_cast<size_t>(ready) * rw * 4);
    S.out.d2h += static_cast<int64_t>(ready) * rw * 4;
    S.tail += ready;
    if (!final) {
        *S.h_tail.p = S.tail;
        LABS_CUDA(cudaMemcpyAsync(S.ctr.p + 2, S.h_tail.p, sizeof(unsigned long long),
                                  cudaMemcpyHostToDevice, st));
        LABS_CUDA(cudaStreamSynchronize(st));
        S.out.h2d += 8;
        ++S.out.ring_drains;
    }
}

void DeviceRunner::poll(int s) {
    Slot& S = slot_[s];
    if (!S.busy) return;
    LABS_CUDA(cudaMemcpyAsync(S.h_head.p, S.ctr.p, sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, drain_st_));
    LABS_CUDA(cudaStreamSynchronize(drain_st_));
    const unsigned long long head = *S.h_head.p;
    if (head - S.tail >= static_cast<unsigned long long>(ring_slots) / 4) drain(S, head, false);
}

JobOut DeviceRunner::finish(int s) {
    Slot& S = slot_[s];
    LABS_CUDA(cudaEventSynchronize(S.ev_done));
    const unsigned long long head = S.h_ctr.p[0];
    const int* ctl = reinterpret_cast<const int*>(S.h_ctr.p + 3);
    S.busy = false;
    if (ctl[0] & 2) throw CudaFailure("shared-memory bounds check failed (LABS_BOUNDS_CHECK build)");
    if (ctl[0]) throw CudaFailure("record ring drain stalled (no host drain for 20 s)");
    drain(S, head, true);
    S.seq0 += head;
    JobOut out = std::move(S.out);
    out.nrec = static_cast<int64_t>(head);
    out.stats.resize(static_cast<size_t>(S.nwalks) * kWalkStatWords);
    if (S.nwalks > 0) std::memcpy(out.stats.data(), S.h_stats.p, out.stats.size() * 8);
    out.d2h += static_cast<int64_t>(4 * sizeof(unsigned long long) + out.stats.size() * 8);
    float ms = 0;
    LABS_CUDA(cudaEventElapsedTime(&ms, S.ev_k0, S.ev_k1));
    out.kernel_ms = ms;
    if (S.seeded) {
        LABS_CUDA(cudaEventElapsedTime(&ms, S.seed_from, S.seed_to));
        out.seed_ms = ms;
    }
    if (!out.cancelled) out.group(wp.rec_words);
    return out;
}

JobOut DeviceRunner::run_sync(const Job& job) {
    LABS_CUDA(cudaSetDevice(dev));
    launch(0, job);
    while (!done(0)) {
        poll(0);
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    return finish(0);
}

// ------------------------------------------------------------------ Executor
void Executor::start() {
    started_ = true;
    th_ = std::thread([this] { body(); });
}

void Executor::push(Job job) {
    {
        std::lock_guard<std::mutex> lock(mu_);
        in_.push_back(std::move(job));
        ++pushed_;
    }
    cv_.notify_all();
}

JobOut Executor::pop() {
    std::unique_lock<std::mutex> lock(mu_);
    cv_.wait(lock, [&] { return !out_.empty() || failed_; });
    if (out_.empty()) throw CudaFailure(err_);
    JobOut o = std::move(out_.front());
    out_.pop_front();
    ++popped_;
    return o;
}

void Executor::cancel() {
    {
        std::lock_guard<std::mutex> lock(mu_);
        cancel_ = true;
    }
    cv_.notify_all();
}

void Executor::stop() {
    if (!started_) return;
    {
        std::lock_guard<std::mutex> lock(mu_);
        closed_ = true;
    }
    cv_.notify_all();
    if (th_.joinable()) th_.join();
    started_ = false;
}

void Executor::body() {
    std::deque<int> inflight;  // slots in launch order
    const bool timing = std::getenv("LABS_TIMING") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const auto ms = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    try {
        LABS_CUDA(cudaSetDevice(dr_.dev));
        auto last_poll = std::chrono::steady_clock::now();
        for (;;) {
            Job job;
            bool have = false, cancel = false;
            {
                std::unique_lock<std::mutex> lock(mu_);
                cancel = cancel_;
                if (cancel) in_.clear();
                if (inflight.size() < 2 && !in_.empty() &&
                    (inflight.empty() || dr_.fits(1 - inflight.back(), in_.front()))) {
                    job = std::move(in_.front());
                    in_.pop_front();
                    have = true;
                } else if (inflight.empty()) {
                    if (closed_ || cancel) break;
                    cv_.wait(lock, [&] { return !in_.empty() || closed_ || cancel_; });
                    continue;
                }
            }
            if (have) {
                const int s = inflight.empty() ? 0 : 1 - inflight.back();
                if (timing)
                    std::fprintf(stderr, "[labs] dev %d t=%.2f ms launch %lld walks on slot %d\n", dr_.dev,
                                 ms(), static_cast<long long>(job.nwalks), s);
                const double tl = ms();
                dr_.launch(s, job);
                if (timing && ms() - tl > 1.0)
                    std::fprintf(stderr, "[labs] dev %d launch call took %.2f ms\n", dr_.dev, ms() - tl);
                inflight.push_back(s);
                continue;
            }
            if (cancel)
                for (int s : inflight) dr_.cancel(s);
            const int s0 = inflight.front();
            if (dr_.done(s0)) {
                const double tf = ms();
                JobOut o = dr_.finish(s0);
                if (timing && ms() - tf > 1.0)
                    std::fprintf(stderr, "[labs] dev %d finish call took %.2f ms\n", dr_.dev, ms() - tf);
                if (timing)
                    std::fprintf(stderr, "[labs] dev %d t=%.2f ms done slot %d (kernel %.2f ms, seed %.2f ms, "
                                 "%lld records, %lld ring drains)\n", dr_.dev, ms(), s0, o.kernel_ms,
                                 o.seed_ms, static_cast<long long>(o.nrec),
                                 static_cast<long long>(o.ring_drains));
                inflight.pop_front();
                {
                    std::lock_guard<std::mutex> lock(mu_);
                    out_.push_back(std::move(o));
                }
                cv_.notify_all();
                continue;
            }
            const auto now = std::chrono::steady_clock::now();
            if (now - last_poll > std::chrono::microseconds(500)) {
                const double tp = ms();
                for (int s : inflight) dr_.poll(s);
                if (timing && ms() - tp > 1.0)
                    std::fprintf(stderr, "[labs] dev %d poll took %.2f ms\n", dr_.dev, ms() - tp);
                last_poll = now;
            }
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    } catch (const std::exception& e) {
        // (a failed device may leave launches in flight; the runner is dropped by the caller)
        std::lock_guard<std::mutex> lock(mu_);
        err_ = e.what();
        failed_ = true;
    }
    cv_.notify_all();
}

}  // namespace labs_b200
