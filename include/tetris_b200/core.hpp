// tetris_b200 — B200-native drop-in for the reference's RNS-CKKS evaluation
// path. Core layer: word arithmetic / RNG / errors (reference common.hpp) and
// the ring layer (reference ring.hpp) with DEVICE-resident polynomials.
//
// Same class and function names as namespace tetris:: so that switching a
// caller is `#include "tetris_b200/tetris.hpp"` + `namespace tetris_b200`.
// Host-side producers (RNG, prime search, NTT table construction, samplers)
// run on the CPU exactly as the reference does, so keys, ciphertexts and
// tables are bit-identical; all polynomial arithmetic runs on the GPU through
// the C-ABI in include/tetris_b200.h. There is no CPU fallback: every
// arithmetic call fails with TetrisError("gpu", ...) when no device exists.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "tetris_b200.h"

namespace tetris_b200 {

using u16 = uint16_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i64 = int64_t;
using u128 = unsigned __int128;
using i128 = __int128;

// ---------------------------------------------------------------------------
// Errors (reference common.hpp:216-224): "[tag] message"
// ---------------------------------------------------------------------------
class TetrisError : public std::runtime_error {
public:
    TetrisError(const std::string& tag, const std::string& what)
        : std::runtime_error("[" + tag + "] " + what), tag_(tag) {}
    const std::string& tag() const { return tag_; }

private:
    std::string tag_;
};

// Throws TetrisError for a failed C-ABI call (tag from the "[tag]" prefix).
void check_tg(int rc);

// ---------------------------------------------------------------------------
// Host word arithmetic (reference common.hpp:24-97)
// ---------------------------------------------------------------------------
inline u64 add_mod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
inline u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : q - (b - a); }
inline u64 neg_mod(u64 a, u64 q) { return a ? q - a : 0; }
inline u64 mul_mod(u64 a, u64 b, u64 q) { return u64((u128(a) * u128(b)) % u128(q)); }
inline u64 shoup_precompute(u64 w, u64 q) { return u64((u128(w) << 64) / q); }
inline u64 mul_mod_shoup(u64 a, u64 w, u64 ws, u64 q) {
    u64 r = a * w - u64((u128(a) * ws) >> 64) * q;
    return r < q ? r : r - q;
}
u64 pow_mod(u64 base, u64 exp, u64 q);
u64 inv_mod(u64 a, u64 q);
inline i64 to_centered(u64 x, u64 q) { return x <= q / 2 ? i64(x) : i64(x) - i64(q); }
inline u64 from_centered(i64 x, u64 q) {
    i64 r = x % i64(q);
    return u64(r < 0 ? r + i64(q) : r);
}
i64 round_half_away(double x);
bool is_prime_u64(u64 n);
std::vector<u64> find_ntt_primes(int bits, std::size_t count, u64 modulus, std::vector<u64> exclude = {});

// ---------------------------------------------------------------------------
// Seeded splittable RNG (reference common.hpp:154-210). Same engine
// (std::mt19937_64 seeded with splitmix64(seed)), same rejection sampler,
// same Box-Muller pairing and split() derivation, so every sample matches.
// ---------------------------------------------------------------------------
u64 splitmix64(u64 x);

class Rng {
public:
    explicit Rng(u64 seed);
    u64 seed() const { return seed_; }
    u64 next() { return eng_(); }
    u64 uniform(u64 bound);
    double normal();
    Rng split(u64 label) const;

private:
    u64 seed_;
    std::mt19937_64 eng_;
    bool spare_ok_ = false;
    double spare_ = 0.0;
};

// ---------------------------------------------------------------------------
// Ring layer
// ---------------------------------------------------------------------------
enum class Form { coeff, eval };

struct NoiseParams {
    double gaussian_sigma = 3.2;
    u32 secret_hamming_weight = 0;
};

// Host copy of the per-modulus NTT tables (reference ring.hpp:15-51); built
// with the reference's psi search so they are canonical per modulus.
struct NttTables {
    u64 q = 0, psi = 0;
    std::vector<u64> w, w_shoup, winv, winv_shoup;
    u64 n_inv = 0, n_inv_shoup = 0;
    void init(u64 modulus, u32 degree, Rng& rng);
};

// Device context + stream of one ring. Shared by the ring and every device
// buffer allocated on it, so buffers may safely outlive their RingParams.
struct DeviceState {
    tg_context* ctx = nullptr;
    void* stream = nullptr;
    std::mutex mu;
    std::vector<void*> workers;  // extra streams for concurrent pipelines
    DeviceState() = default;
    DeviceState(const DeviceState&) = delete;
    DeviceState& operator=(const DeviceState&) = delete;
    ~DeviceState();
    void* worker_stream(std::size_t i);
};

// Routes every device call the current host thread makes on `ring` to
// `stream` for the scope's lifetime (one stream per host thread when
// independent ciphertexts run concurrently, the reference's thread-pool
// granularity, protocol.hpp:297-311).
class RingParams;
class StreamScope {
public:
    StreamScope(const RingParams& ring, void* stream);
    ~StreamScope();
    StreamScope(const StreamScope&) = delete;
    StreamScope& operator=(const StreamScope&) = delete;

private:
    const void* prev_state_;
    void* prev_stream_;
};

// Per-process default CUDA device for new contexts (torchrun: LOCAL_RANK).
void set_default_device(int device);
int default_device();

// Replaces reference RingParams (ring.hpp:116-195). Immutable after
// construction; the device context (tables in HBM, a stream, a memory pool)
// is created on first device use.
class RingParams {
public:
    RingParams(u32 degree, std::vector<u64> moduli, u32 special_count);
    ~RingParams();
    RingParams(const RingParams&) = delete;
    RingParams& operator=(const RingParams&) = delete;

    u32 degree() const { return degree_; }
    u32 log_degree() const { return log_degree_; }
    const std::vector<u64>& moduli() const { return moduli_; }
    u32 special_count() const { return special_count_; }
    u32 q_count() const { return u32(moduli_.size()) - special_count_; }
    int max_level() const { return int(q_count()) - 1; }
    u64 modulus(u32 idx) const { return moduli_[idx]; }
    const NttTables& tables(u32 idx) const { return tables_[idx]; }
    u32 eval_exp(u32 slot) const { return eval_exp_[slot]; }
    u32 slot_of_exp(u32 exp) const { return slot_of_exp_[exp]; }
    const std::vector<u32>& eval_exp_table() const { return eval_exp_; }
    const std::vector<u32>& slot_of_exp_table() const { return slot_of_exp_; }
    double total_log2_q(int level) const;
    bool compatible(const RingParams& other) const { return this == &other; }

    // Device side (lazy).
    tg_context* dev() const;
    void* stream() const;  // cudaStream_t of this ring's work
    const std::shared_ptr<DeviceState>& device_state() const;
    void synchronize() const;
    int device() const { return device_; }

private:
    void build_eval_order_map();
    u32 degree_, log_degree_;
    std::vector<u64> moduli_;
    u32 special_count_;
    std::vector<NttTables> tables_;
    std::vector<u32> eval_exp_, slot_of_exp_;
    int device_;
    mutable std::once_flag dev_once_;
    mutable std::shared_ptr<DeviceState> dev_;
};

// Device buffer (stream-ordered pool allocation on the ring's stream).
class DeviceBuffer {
public:
    DeviceBuffer(const RingParams& ring, std::size_t words);
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    u64* data() const { return ptr_; }
    std::size_t words() const { return words_; }

    // Memoised forward transforms of (immutable, shared) contents: the eval
    // form of the `nparts` polys of shape (level, nspecial) starting at `off`.
    // Ladder operands are multiplied several times (and squared), so each is
    // transformed once. Bit-exact: the NTT is deterministic.
    struct EvalCache {
        std::size_t off;
        int level, nspecial, nparts;
        void* stream;
        std::shared_ptr<DeviceBuffer> buf;
    };
    std::shared_ptr<DeviceBuffer> find_eval(std::size_t off, int level, int nspecial, int nparts, void* stream) const;
    void put_eval(std::size_t off, int level, int nspecial, int nparts, void* stream,
                  std::shared_ptr<DeviceBuffer> buf) const;
    // contents are about to be overwritten (reused upload buffers)
    void clear_eval_cache() const;

private:
    std::shared_ptr<DeviceState> dev_;
    void* stream_ = nullptr;  // allocation stream
    mutable std::mutex cache_mu_;
    mutable std::vector<EvalCache> cache_;
    u64* ptr_ = nullptr;
    std::size_t words_ = 0;
};

// Replaces reference Poly (ring.hpp:204-374): rows 0..level over the q-chain
// plus nspecial special rows, row-major, resident in HBM. Copies are cheap
// handles; mutation is copy-on-write, so value semantics match the reference.
class Poly {
public:
    Poly() = default;
    Poly(const RingParams& ring, int level, Form form, int nspecial = 0);  // zero-filled

    const RingParams& ring() const { return *ring_; }
    int level() const { return level_; }
    int nspecial() const { return nspecial_; }
    Form form() const { return form_; }
    void set_form(Form f) { form_ = f; }
    int rows() const { return level_ + 1 + nspecial_; }
    bool empty() const { return ring_ == nullptr; }
    std::size_t words() const { return std::size_t(rows()) * ring_->degree(); }
    u32 modulus_index(int r) const { return r <= level_ ? u32(r) : ring_->q_count() + u32(r - level_ - 1); }
    u64 row_modulus(int r) const { return ring_->modulus(modulus_index(r)); }

    // device data (const: shared; mutable: made unique first)
    const u64* data() const { return st_->data() + off_; }
    u64* mutable_data();
    bool shares_storage_with(const Poly& o) const { return st_ == o.st_; }
    const std::shared_ptr<DeviceBuffer>& storage() const { return st_; }
    std::size_t offset() const { return off_; }

    // host transfer
    std::vector<u64> to_host() const;
    void to_host(u64* dst) const;
    static Poly from_host(const RingParams& ring, const u64* src, int level, Form form, int nspecial = 0);
    static Poly from_host(const RingParams& ring, const std::vector<u64>& src, int level, Form form, int nspecial = 0);

    // transforms (ring.hpp:234-246)
    void ntt_forward();
    void ntt_inverse();
    // element-wise (ring.hpp:250-325)
    void add_inplace(const Poly& o);
    void sub_inplace(const Poly& o);
    void negate_inplace();
    void mul_pointwise_inplace(const Poly& o);
    void mul_acc_pointwise(const Poly& x, const Poly& y);
    void mul_scalar_inplace(const std::vector<u64>& scalar_per_modulus);
    void mul_small_scalar_inplace(u64 s);
    // structural (ring.hpp:329-340)
    void drop_to_level(int new_level);
    void drop_special();
    void check_shape(const Poly& o) const;

    // internal: a view of `rows` rows of an existing buffer
    static Poly view(const RingParams& ring, std::shared_ptr<DeviceBuffer> st, std::size_t off, int level, Form form,
                     int nspecial);

private:
    const RingParams* ring_ = nullptr;
    int level_ = 0;
    int nspecial_ = 0;
    Form form_ = Form::coeff;
    std::shared_ptr<DeviceBuffer> st_;
    std::size_t off_ = 0;
};

// Free ring operations (ring.hpp:380-518)
Poly poly_add(const Poly& a, const Poly& b);
Poly poly_sub(const Poly& a, const Poly& b);
Poly ntt_transform(const Poly& p, Form target);
Poly poly_mul(const Poly& a, const Poly& b);
Poly automorphism_apply(const Poly& p, u64 exponent);
Poly rescale_round(const Poly& p);
// Poly::mul_monomial (ring.hpp:343-361): X^e * p, coefficient form.
Poly mul_monomial(const Poly& p, u32 e);
// raise_level (ring.hpp:523-545): a level-0 coefficient poly lifted to
// (new_level, nspecial) as the centered integer mod q0.
Poly raise_level(const Poly& p, int new_level, int nspecial = 0);

// Samplers: drawn on the host from the same streams as the reference
// (ring.hpp:442-487), then uploaded.
Poly sample_uniform(const RingParams& ring, int level, int nspecial, Rng& rng);
Poly poly_from_i64(const RingParams& ring, const std::vector<i64>& coeffs, int level, int nspecial = 0);
Poly sample_gaussian(const RingParams& ring, double sigma, int level, int nspecial, Rng& rng);
Poly sample_ternary_hw(const RingParams& ring, u32 h, int level, int nspecial, Rng& rng);
// host-only helpers (unit tests of the samplers without a device)
std::vector<u64> sample_uniform_host(const RingParams& ring, int level, int nspecial, Rng& rng);
std::vector<i64> sample_gaussian_coeffs(u32 n, double sigma, Rng& rng);
std::vector<i64> sample_ternary_coeffs(u32 n, u32 h, Rng& rng);

}  // namespace tetris_b200
