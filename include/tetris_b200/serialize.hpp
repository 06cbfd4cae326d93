// Wire formats of the evaluation path (reference serialize.hpp:13-353):
// little-endian, self-describing { magic "TTRS", version, kind, ring geometry }
// objects, byte-identical to the reference's writer, so scientist artifacts
// load straight onto the GPU. Switching keys are seed-compressed: only the
// b-parts travel; the a-parts are regenerated from a_seed (mt19937_64 streams
// on the host, the same as keygen) and transformed on the device.
// SURVEY 8(f) rank 3. Repack keys / eval key sets / queries belong to the
// out-of-scope PFE/repack stages and are not handled here.
#pragma once

#include <cstdint>
#include <vector>

#include "tetris_b200/evaluator.hpp"

namespace tetris_b200 {

enum class ObjectKind : u16 {
    ciphertext = 1,
    switching_key = 2,
    repack_keys = 3,
    eval_keyset = 4,
    query = 5,
    chain = 6,
    secret_key = 7,
};

std::vector<uint8_t> serialize_ciphertext(const Ciphertext& ct);
Ciphertext deserialize_ciphertext(const std::vector<uint8_t>& buf, const RingParams& ring);
std::size_t ciphertext_size(const RingParams& ring, int level, u32 parts = 2);

std::vector<uint8_t> serialize_switching_key(const SwitchingKey& k);
SwitchingKey deserialize_switching_key(const std::vector<uint8_t>& buf, const RingParams& ring);

std::vector<uint8_t> serialize_chain(const MinimaxChain& c);
MinimaxChain deserialize_chain(const std::vector<uint8_t>& buf);

std::vector<uint8_t> serialize_secret_key(const SecretKey& sk);
SecretKey deserialize_secret_key(const std::vector<uint8_t>& buf, const RingParams& ring);

}  // namespace tetris_b200
