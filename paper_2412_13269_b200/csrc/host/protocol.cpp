// Device composition of explore_from_repacked (reference protocol.hpp:241-328).
//
// B200-first structure, same results: the reference runs merge -> Half-BTS ->
// two local thresholds per group on a host thread pool; here every group's
// merge and Half-BTS issue on the device in turn, and then ALL 2 x groups
// local-threshold inputs (left and right halves of every group) run through
// eval_private_threshold as ONE ciphertext batch (one launch per op, the
// relinearisation / rotation keys read once for the whole batch). A batch is
// exactly its independent members, and the mod-q sums afterwards are exact,
// so the count ciphertext is residue-identical to the reference's
// (tests/test_gpu_protocol.py).
#include "internal.hpp"
#include "tetris_b200/protocol.hpp"

namespace tetris_b200 {

Ciphertext explore_from_repacked(const KeyContext& ctx_big, const Evaluator& ev, const BootstrapEvaluator& bts,
                                 const MinimaxChain& chain_local, const MinimaxChain& chain_global,
                                 const std::vector<Ciphertext>& repacked, std::size_t p_total, const Ciphertext& t0,
                                 const Ciphertext& t1, const Ciphertext& norm, u64 small_sk_id,
                                 const ExploreKeys& keys) {
    if (!keys.merge || !keys.big) throw TetrisError("protocol", "explore needs the merge and big-ring keys");
    if (repacked.empty()) throw TetrisError("protocol", "nothing to merge");
    const u32 n_big = ctx_big.ring().degree(), n_small = repacked[0].ring().degree();
    if (n_small == 0 || n_big % n_small != 0) throw TetrisError("protocol", "ring degrees do not nest");
    const u32 arity = n_big / n_small;
    const std::size_t groups = (repacked.size() + arity - 1) / arity;
    for (const auto& ct : repacked)
        if (ct.sk_id != small_sk_id) throw TetrisError("protocol", "repacked ciphertexts under a foreign key");

    // lines 8-9: merge `arity` repacked ciphertexts per big-ring ciphertext,
    // then Half-BTS (its two EvalMod halves already run as one batch)
    std::vector<Ciphertext> halves;
    halves.reserve(2 * groups);
    for (std::size_t g = 0; g < groups; ++g) {
        std::vector<const Ciphertext*> batch(arity, nullptr);
        for (u32 k = 0; k < arity; ++k)
            if (g * arity + k < repacked.size()) batch[k] = &repacked[g * arity + k];
        auto [l, r] = bts.half_bts(ev, ring_merge_many(ctx_big, batch, *keys.merge), *keys.big);
        halves.push_back(std::move(l));
        halves.push_back(std::move(r));
    }
    // lines 10-11: the local threshold on every half, as one batch
    const std::size_t B = halves.size();
    std::vector<Ciphertext> bits = B == 1 ? std::vector<Ciphertext>{eval_private_threshold(
                                               ev, halves[0], t0, norm, chain_local, *keys.big)}
                                          : unstack_ciphertext(eval_private_threshold(
                                                ev, stack_ciphertexts(halves), stack_ciphertexts(std::vector<Ciphertext>(B, t0)),
                                                stack_ciphertexts(std::vector<Ciphertext>(B, norm)), chain_local,
                                                *keys.big));
    // lines 12-13: per group left + right, then the groups in order
    Ciphertext score = bits[0];
    score.add_inplace(bits[1]);
    for (std::size_t g = 1; g < groups; ++g) {
        Ciphertext part = bits[2 * g];
        part.add_inplace(bits[2 * g + 1]);
        score.add_inplace(part);
    }
    // lines 14-16: slot sum, then the global threshold with the 1/p normaliser
    Ciphertext summed = inner_sum(ev, score, n_big / 2, *keys.big);
    return eval_private_threshold_plain_norm(ev, summed, t1, 1.0 / double(p_total), chain_global, *keys.big);
}

}  // namespace tetris_b200
