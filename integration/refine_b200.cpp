// refine_b200.cpp -- Step 2 (refine, pq.cpp:114-176) scored through the GPU
// neighbourhood kernel K5 (labs_pq_score), linked in place of the reference's CPU refine
// (integration/Makefile weakens the `refine` symbol of the reference's pq.o, so this
// definition wins the link and the reference's refine_with_operators, pq.cpp:203-228, calls it).
//
// The frontier is the reference's own SearchFrontier (pq.hpp:37-70, pq.cpp:33-49) and its
// operations run in exactly the reference order -- pop the pivot, then for i = 0..L-1:
// seen? -> mark -> push the flip neighbour -> improvement check -> the T_r left and T_r
// right rotations (seen? -> mark -> push) -- so the refinement trajectory is identical.
// Only the arithmetic moves to the GPU: one labs_pq_score launch per pivot returns every
// flip delta, rotation energy and rotation hash the loop consumes, replacing the O(L^2)
// CorrelationState construction and the ~(1 + 2 T_r) O(L) updates per neighbour.
#include <algorithm>
#include <chrono>
#include <stdexcept>
#include <unordered_set>
#include <vector>

#include "labs/pq.hpp"
#include "labs_gpu.h"

namespace labsearch {

RefineResult refine(const Candidate& start, const PqConfig& config) {
    const int n = start.seq.length();
    config.validate(n);
    const long long t_u = config.effective_stale_limit(n);
    const int t_r = std::min(config.max_rotation, n - 1);  // rotations need T_r < L
    const auto& tab = TabulationHash::instance();

    const bool has_deadline = config.deadline_s > 0;
    const auto deadline = std::chrono::steady_clock::now() +
                          std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                              std::chrono::duration<double>(config.deadline_s));

    RefineResult res{start, 0, 0, 0, false, {}};
    Energy e_best = start.energy;

    SearchFrontier frontier(config.queue_capacity);
    frontier.mark(start.seq.canonical_hash(0));
    frontier.push(start.seq, start.energy);
    ++res.pushes;

    const int nrot = t_r > 0 ? t_r : 0;
    std::vector<std::int32_t> delta(static_cast<std::size_t>(n));
    std::vector<std::int32_t> rot_e(static_cast<std::size_t>(n) * 2 * std::max(nrot, 1));
    std::vector<std::uint64_t> rot_h(rot_e.size());
    std::vector<Sign> rot(static_cast<std::size_t>(n));

    long long u = 0;
    while (u < t_u && !frontier.empty()) {
        if (has_deadline && std::chrono::steady_clock::now() >= deadline) break;
        ++u;
        ++res.pivots;
        auto entry = frontier.pop_min();
        BinarySequence seq = entry.seq.unpack();
        std::int64_t e64 = 0;
        const int rc = labs_pq_score(n, nrot, seq.data(), delta.data(), rot_e.data(),
                                     rot_h.data(), &e64);
        if (rc == LABS_EINVAL) throw std::invalid_argument(labs_last_error());
        if (rc != LABS_OK) throw std::runtime_error(labs_last_error());
        const Energy e = e64;
        if (config.debug_check_energy && e != entry.energy)
            throw std::logic_error("pq frontier energy bookkeeping diverged");
        if (e < e_best) {  // rotation-pushed pivots bypass the neighbour check (pq.cpp:146-153)
            e_best = e;
            res.best = Candidate{seq, e, Origin::dfs, start.prefix};
            ++res.improvements;
            res.improvement_log.emplace_back(res.pivots, e_best);
            u = 0;
        }
        const std::uint64_t h = seq.canonical_hash(0);

        for (int i = 0; i < n; ++i) {
            const std::uint64_t nh = h ^ tab.flip_mask(i, 0);
            if (frontier.seen(nh)) continue;
            const Energy d = delta[static_cast<std::size_t>(i)];
            seq.flip(i);  // seq is now the neighbour
            frontier.mark(nh);
            if (frontier.push(seq, e + d)) ++res.pushes;
            if (e + d < e_best) {
                e_best = e + d;
                res.best = Candidate{seq, e_best, Origin::dfs, start.prefix};
                ++res.improvements;
                res.improvement_log.emplace_back(res.pivots, e_best);
                u = 0;
            }
            // make_rotations (pq.cpp:103-112): left chain, then right chain
            for (int dir = 0; dir < 2 && nrot > 0; ++dir) {
                for (int r = 1; r <= nrot; ++r) {
                    const std::size_t o = (static_cast<std::size_t>(i) * 2 + dir) * nrot + (r - 1);
                    const std::uint64_t hr = rot_h[o];
                    if (frontier.seen(hr)) continue;
                    frontier.mark(hr);
                    const Sign* x = seq.data();  // left: v_j = x_{j+r}; right: v_j = x_{j-r}
                    std::rotate_copy(x, x + (dir == 0 ? r : n - r), x + n, rot.begin());
                    frontier.push(BinarySequence(rot), rot_e[o]);
                }
            }
            seq.flip(i);  // restore the pivot
        }
    }
    res.queue_exhausted = frontier.empty();
    return res;
}

}  // namespace labsearch
