// runner.hpp -- per-device execution of Step-1 walk jobs (host side of K3 + K1 + K2).
//
// A job is a batch of walks -- restart ranges of walkers, in the reference's order -- that
// one device seeds (K3, generator streams kept on the device between jobs), walks (K1) and
// compacts (K2: the sieve's record ring).  A DeviceRunner owns the device tables and two
// slots (stream + buffers), so two jobs overlap; an Executor thread per device feeds the
// slots from a job queue, drains each slot's record ring with async copies while its launch
// runs, and hands finished jobs back in order.  engine.cpp schedules jobs and replays their
// results through the reference's sink chain (saw.cpp:173-194, candidate.hpp:84-99).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host_util.hpp"

namespace labs_b200 {

struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define LABS_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess) {                                                           \
            throw ::labs_b200::CudaFailure(std::string(#call) + ": " + cudaGetErrorString(_e)); \
        }                                                                                  \
    } while (0)

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
    void reserve(size_t count) {  // grow-only (geometric); contents are not preserved
        if (count <= n) return;
        count = std::max(count, 2 * n);  // (growing batches would reallocate every time)
        release();
        LABS_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
    }
};

// Grow-only pinned host staging (async H2D of job tables, D2H drains).
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
    void reserve(size_t count) {  // grow-only (geometric)
        if (count <= n) return;
        count = std::max(count, 2 * n);
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        LABS_CUDA(cudaMallocHost(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
    }
};

// Restarts [r0, r1) of one walker, drawn in order from its stream (walker_loop,
// saw.cpp:196-214).  `gen` is the walker's generator slot on its device: restart r0 > 0
// continues the stream the walker's previous segment left there.
struct Segment {
    uint32_t walker;
    int64_t r0, r1;
    uint32_t gen = 0;
};

struct WalkRecordView {
    int64_t walk;        // job-local walk index
    int64_t iteration;
    int64_t energy;
    uint64_t hash;       // canonical_hash(0) of the full sequence (computed on the device)
    const uint32_t* half;
};

struct Job {
    std::vector<Segment> segs;
    int64_t nwalks = 0;
    // >= 0: the walks' initial halves were seeded ahead (DeviceRunner::preseed) and start at
    // this walk of the runner's pool buffer: no K3 in this job's launch
    int64_t pool_off = -1;
    // seed-table mode: packed initial halves (nwalks x hw) instead of K3
    const uint32_t* host_halves = nullptr;
    int* score_out = nullptr;  // labs_skew_flip_deltas: deltas / correlations of the start
    int* corr_out = nullptr;
};

// A finished job: its sieve records (grouped by walk) and per-walk stats.
struct JobOut {
    std::vector<uint32_t> rec;             // nrec x rec_words, ring order
    int64_t nrec = 0;
    std::vector<int64_t> stats;            // nwalks x kWalkStatWords
    std::vector<uint32_t> walk_walker;     // per job walk: walker, restart
    std::vector<int64_t> walk_restart;
    std::vector<WalkRecordView> views;     // records sorted by (walk, iteration)
    std::vector<int64_t> start;            // views of walk i: [start[i], start[i+1])
    double kernel_ms = 0, seed_ms = 0;
    int64_t h2d = 0, d2h = 0;
    int64_t ring_drains = 0;               // partial drains while the launch ran
    bool cancelled = false;
    void group(int rec_words);
};

// K3 job tables (device + pinned staging): walker, prefix bits, generator slot | restarts,
// first walk | fresh-stream flag, per segment.
struct SeedBufs {
    DevBuf<uint32_t> seg32;
    DevBuf<int64_t> seg64;
    DevBuf<int32_t> seg_init;
    PinnedBuf<uint32_t> h_seg32;
    PinnedBuf<int64_t> h_seg64;
    PinnedBuf<int32_t> h_init;
    bool fits(size_t nseg) const {
        return 3 * nseg <= seg32.n && 2 * nseg <= seg64.n && nseg <= seg_init.n &&
               3 * nseg <= h_seg32.n && 2 * nseg <= h_seg64.n && nseg <= h_init.n;
    }
    void reserve(size_t nseg) {
        h_seg32.reserve(3 * nseg);
        h_seg64.reserve(2 * nseg);
        h_init.reserve(nseg);
        seg32.reserve(3 * nseg);
        seg64.reserve(2 * nseg);
        seg_init.reserve(nseg);
    }
};

class DeviceRunner {
public:
    int dev = 0;
    WalkParams wp{};
    int grid_cap = 0;
    int64_t resident = 0;        // walks resident at once (one wave)
    int64_t ring_slots = 0;      // record ring capacity per slot (power of two)
    uint64_t seed = 0;           // Rng seed of the current pool
    const Derived* d = nullptr;  // prefix bits of the current pool

    ~DeviceRunner();
    void init(int device, const WalkParams& params);
    void reserve_generators(size_t n) { rng.reserve(4 * std::max<size_t>(n, 1)); }

    // Enqueue a job on slot s (K3 unless host halves, then K1, then the stats drain);
    // returns at once.  K3 launches run in job order across the two slots.
    void launch(int s, const Job& job);
    bool fits(int s, const Job& job) const;  // launch(s, job) allocates nothing
    bool done(int s);                   // the slot's launch and drains completed
    void poll(int s);                   // drain the slot's ring if it is filling up
    void cancel(int s);                 // ask the slot's K1 to stop taking walks
    JobOut finish(int s);               // after done(s): final drain, stats, grouping
    JobOut run_sync(const Job& job);    // launch on slot 0 and wait (bench, seed-table mode)
    // Seed the initial halves of a whole (independent) pool in one K3 launch, walks in
    // `segs` order, before any job is pushed; jobs then take slices (Job::pool_off), so no
    // K3 waits behind the other slot's walk blocks at a job boundary.  Idle runner only.
    void preseed(const std::vector<Segment>& segs, int64_t nwalks);
    bool busy(int s) const { return slot_[s].busy; }

private:
    struct Slot {
        cudaStream_t st = nullptr;
        cudaEvent_t ev_s0 = nullptr, ev_s1 = nullptr, ev_k0 = nullptr, ev_k1 = nullptr,
                    ev_done = nullptr;
        DevBuf<uint32_t> halves, ring, tag;
        DevBuf<int64_t> stats;
        DevBuf<unsigned long long> ctr;             // head, walk queue, tail, ctl (2 x int)
        SeedBufs sb;
        PinnedBuf<uint32_t> h_ring, h_tag, h_halves;
        PinnedBuf<int64_t> h_stats;
        PinnedBuf<unsigned long long> h_ctr, h_head, h_tail;
        PinnedBuf<int> h_cancel;
        bool busy = false, seeded = false, cancel_sent = false;
        cudaEvent_t seed_from = nullptr, seed_to = nullptr;  // this job's K3 (seed_ms)
        int64_t nwalks = 0;
        unsigned long long tail = 0;
        unsigned long long seq0 = 0;  // records this slot's ring carried in earlier launches
        JobOut out;
    };
    Slot slot_[2];
    cudaStream_t drain_st_ = nullptr;
    cudaEvent_t last_seed_ = nullptr;   // the latest K3 (the next one waits for it)
    cudaEvent_t pre_ev0_ = nullptr, preseed_ev_ = nullptr;  // the pool's preseed K3 (pool_off
                                                            // jobs wait for preseed_ev_)
    DevBuf<uint64_t> fm, tab, tabfull, rng;
    DevBuf<uint32_t> pool_halves;       // preseeded halves of the current pool
    SeedBufs pool_sb;
    int64_t pool_walks_ = 0, pending_h2d_ = 0;
    bool preseed_timed_ = true;
    void drain(Slot& S, unsigned long long head, bool final);
    // K3 of `segs` into `halves` on stream st (after the previous K3); returns H2D bytes
    int64_t seed_into(cudaStream_t st, SeedBufs& B, const std::vector<Segment>& segs,
                      uint32_t* halves, cudaEvent_t ev0, cudaEvent_t ev1);
};

// One host thread per device: runs queued jobs two at a time on the runner's slots, keeps
// their record rings drained, and returns finished jobs in queue order.
class Executor {
public:
    explicit Executor(DeviceRunner& dr) : dr_(dr) {}
    ~Executor() { stop(); }
    void start();
    void push(Job job);
    JobOut pop();          // blocks; throws CudaFailure if the device thread failed
    void cancel();         // drop queued jobs, stop the running launches early
    void stop();           // close the queue and join (after cancel: discards results)
    int64_t pushed() const { return pushed_; }
    int64_t popped() const { return popped_; }

private:
    void body();
    DeviceRunner& dr_;
    std::thread th_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Job> in_;
    std::deque<JobOut> out_;
    bool closed_ = false, cancel_ = false, failed_ = false, started_ = false;
    std::string err_;
    int64_t pushed_ = 0, popped_ = 0;
};

}  // namespace labs_b200
