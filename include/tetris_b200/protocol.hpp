// The evaluation half of the TETRIS exploration protocol on the device
// (reference protocol.hpp:241-328, Algorithm 2 lines 8-16): merge the
// repacked small-ring ciphertexts into big-ring ciphertexts, Half-BTS each,
// local threshold on both halves, sum, slot sum, global threshold.
// The reference takes a ProtocolContext (profile.hpp:110-190: rings, key
// contexts, evaluator, bootstrapper and the two chains); the drop-in takes
// those members directly, with the same meaning and error behaviour.
#pragma once

#include "tetris_b200/bootstrap.hpp"
#include "tetris_b200/pfe.hpp"

namespace tetris_b200 {

struct ExploreKeys {
    const SwitchingKey* merge = nullptr;  // embedded small secret -> big secret (EvalKeySet::merge)
    const EvalKeys* big = nullptr;        // relinearisation + Galois manifest (EvalKeySet::big)
};

// repacked: small-ring ciphertexts (score_and_repack's output, under
// small_sk_id); t0, norm at the Half-BTS output level, t1 at the level after
// the local threshold (scientist_setup); p_total: rows of the database.
Ciphertext explore_from_repacked(const KeyContext& ctx_big, const Evaluator& ev, const BootstrapEvaluator& bts,
                                 const MinimaxChain& chain_local, const MinimaxChain& chain_global,
                                 const std::vector<Ciphertext>& repacked, std::size_t p_total, const Ciphertext& t0,
                                 const Ciphertext& t1, const Ciphertext& norm, u64 small_sk_id,
                                 const ExploreKeys& keys);

}  // namespace tetris_b200
