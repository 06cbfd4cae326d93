// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Python bindings over the UNMODIFIED TETRIS reference headers
// (/root/reference/proj/include/tetris/*.hpp, included in place, not copied).
// Built by oracle/Makefile into oracle/_ref/tetris_ref<ext>.so. Only tests/,
// __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs import
// it, and only as the checker or the timed CPU baseline.
//
// The Python surface deliberately mirrors the product module
// (paper_2412_13269_b200.tetris): the same class and method names, so one
// parity script can drive both and compare residues.

#include <pybind11/pybind11.h>
#include <pybind11/numpy.h>
#include <pybind11/stl.h>
#include <pybind11/complex.h>

#include <chrono>
#include <thread>
#include <atomic>

#include "tetris/threshold.hpp"
#include "tetris/bootstrap.hpp"
#include "tetris/serialize.hpp"
#include "tetris/protocol.hpp"

namespace py = pybind11;
using namespace tetris;

namespace {

py::array_t<uint64_t> poly_to_numpy(const Poly& p) {
    const u32 n = p.ring().degree();
    py::array_t<uint64_t> out({py::ssize_t(p.rows()), py::ssize_t(n)});
    auto* dst = out.mutable_data();
    for (int r = 0; r < p.rows(); ++r) std::memcpy(dst + size_t(r) * n, p.row(r), n * 8);
    return out;
}

Poly poly_from_numpy(const RingParams& ring, py::array_t<uint64_t, py::array::c_style | py::array::forcecast> a,
                     int level, Form form, int nspecial) {
    Poly p(ring, level, form, nspecial);
    const u32 n = ring.degree();
    if (a.ndim() != 2 || a.shape(0) != p.rows() || a.shape(1) != py::ssize_t(n))
        throw TetrisError("oracle", "poly_from_numpy: shape mismatch");
    for (int r = 0; r < p.rows(); ++r) std::memcpy(p.row(r), a.data() + size_t(r) * n, n * 8);
    return p;
}

template <class T>
py::array_t<T> vec_to_numpy(const std::vector<T>& v) {
    py::array_t<T> out(py::ssize_t(v.size()));
    std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(T));
    return out;
}

}  // namespace

PYBIND11_MODULE(tetris_ref, m) {
    m.doc() = "Compiled TETRIS reference (oracle; test infrastructure only)";
    m.attr("IMPL") = "reference";

    py::register_exception<TetrisError>(m, "TetrisError", PyExc_RuntimeError);

    py::enum_<Form>(m, "Form").value("coeff", Form::coeff).value("eval", Form::eval);
    py::enum_<Domain>(m, "Domain").value("coeffs", Domain::coeffs).value("slots", Domain::slots);

    m.def("find_ntt_primes", &find_ntt_primes, py::arg("bits"), py::arg("count"), py::arg("modulus"),
          py::arg("exclude") = std::vector<u64>{});
    m.def("round_half_away", &round_half_away);

    py::class_<Rng>(m, "Rng")
        .def(py::init<u64>())
        .def("seed", &Rng::seed)
        .def("next", &Rng::next)
        .def("uniform", &Rng::uniform)
        .def("normal", &Rng::normal)
        .def("split", &Rng::split);

    py::class_<RingParams, std::shared_ptr<RingParams>>(m, "RingParams")
        .def(py::init<u32, std::vector<u64>, u32>())
        .def("degree", &RingParams::degree)
        .def("moduli", &RingParams::moduli)
        .def("special_count", &RingParams::special_count)
        .def("q_count", &RingParams::q_count)
        .def("max_level", &RingParams::max_level)
        .def("modulus", &RingParams::modulus)
        .def("tables", [](const RingParams& r, u32 i) {
            const NttTables& t = r.tables(i);
            py::dict d;
            d["q"] = t.q;
            d["psi"] = t.psi;
            d["w"] = vec_to_numpy(t.w);
            d["w_shoup"] = vec_to_numpy(t.w_shoup);
            d["winv"] = vec_to_numpy(t.winv);
            d["winv_shoup"] = vec_to_numpy(t.winv_shoup);
            d["n_inv"] = t.n_inv;
            d["n_inv_shoup"] = t.n_inv_shoup;
            return d;
        })
        .def("eval_exp_table", [](const RingParams& r) {
            std::vector<u32> v(r.degree());
            for (u32 j = 0; j < r.degree(); ++j) v[j] = r.eval_exp(j);
            return vec_to_numpy(v);
        })
        .def("slot_of_exp_table", [](const RingParams& r) {
            std::vector<u32> v(2 * r.degree());
            for (u32 e = 0; e < 2 * r.degree(); ++e) v[e] = r.slot_of_exp(e);
            return vec_to_numpy(v);
        });

    py::class_<Poly>(m, "Poly")
        .def(py::init<const RingParams&, int, Form, int>(), py::arg("ring"), py::arg("level"),
             py::arg("form"), py::arg("nspecial") = 0, py::keep_alive<1, 2>())
        .def("level", &Poly::level)
        .def("nspecial", &Poly::nspecial)
        .def("form", &Poly::form)
        .def("rows", &Poly::rows)
        .def("to_numpy", &poly_to_numpy)
        .def_static("from_numpy", &poly_from_numpy, py::arg("ring"), py::arg("data"), py::arg("level"),
                    py::arg("form"), py::arg("nspecial") = 0, py::keep_alive<0, 1>())
        .def("copy", [](const Poly& p) { return Poly(p); })
        .def("ntt_forward", &Poly::ntt_forward, py::call_guard<py::gil_scoped_release>())
        .def("ntt_inverse", &Poly::ntt_inverse, py::call_guard<py::gil_scoped_release>())
        .def("mul_monomial", &Poly::mul_monomial)
        .def("add_inplace", &Poly::add_inplace)
        .def("sub_inplace", &Poly::sub_inplace)
        .def("negate_inplace", &Poly::negate_inplace)
        .def("mul_pointwise_inplace", &Poly::mul_pointwise_inplace)
        .def("mul_acc_pointwise", &Poly::mul_acc_pointwise)
        .def("mul_scalar_inplace", &Poly::mul_scalar_inplace)
        .def("mul_small_scalar_inplace", &Poly::mul_small_scalar_inplace)
        .def("drop_to_level", &Poly::drop_to_level);

    m.def("ntt_transform", &ntt_transform, py::call_guard<py::gil_scoped_release>());
    m.def("poly_from_i64", &poly_from_i64, py::arg("ring"), py::arg("coeffs"), py::arg("level"),
          py::arg("nspecial") = 0);
    m.def("raise_level", &raise_level, py::arg("p"), py::arg("new_level"), py::arg("nspecial") = 0);
    m.def("automorphism_apply", &automorphism_apply);
    m.def("rescale_round", &rescale_round);
    m.def("sample_uniform", &sample_uniform, py::keep_alive<0, 1>());
    m.def("sample_gaussian", &sample_gaussian, py::keep_alive<0, 1>());
    m.def("sample_ternary_hw", &sample_ternary_hw, py::keep_alive<0, 1>());

    py::class_<NoiseParams>(m, "NoiseParams")
        .def(py::init([](double sigma, u32 h) { return NoiseParams{sigma, h}; }),
             py::arg("gaussian_sigma") = 3.2, py::arg("secret_hamming_weight") = 0)
        .def_readwrite("gaussian_sigma", &NoiseParams::gaussian_sigma)
        .def_readwrite("secret_hamming_weight", &NoiseParams::secret_hamming_weight);

    py::class_<GadgetVector>(m, "GadgetVector")
        .def(py::init([](u32 g, u32 b) { return GadgetVector{g, b}; }), py::arg("group_size") = 1,
             py::arg("base2_bits") = 0)
        .def_readwrite("group_size", &GadgetVector::group_size)
        .def_readwrite("base2_bits", &GadgetVector::base2_bits);

    py::class_<SecretKey>(m, "SecretKey")
        .def("id", &SecretKey::id)
        .def("coeffs", &SecretKey::coeffs)
        .def("hamming_weight", &SecretKey::hamming_weight)
        .def("shaped", &SecretKey::shaped);
    py::class_<PublicKey>(m, "PublicKey")
        .def_readonly("b", &PublicKey::b)
        .def_readonly("a", &PublicKey::a)
        .def_readonly("sk_id", &PublicKey::sk_id);

    py::class_<Ciphertext>(m, "Ciphertext")
        .def(py::init<>())
        .def_readwrite("parts", &Ciphertext::parts)
        .def_readwrite("scale", &Ciphertext::scale)
        .def_readwrite("domain", &Ciphertext::domain)
        .def_readwrite("sk_id", &Ciphertext::sk_id)
        .def_readwrite("noise_bound", &Ciphertext::noise_bound)
        .def("level", &Ciphertext::level)
        .def("form", &Ciphertext::form)
        .def("degree", &Ciphertext::degree)
        .def("copy", [](const Ciphertext& c) { return Ciphertext(c); })
        .def("to_coeff", &Ciphertext::to_coeff)
        .def("to_eval", &Ciphertext::to_eval)
        .def("drop_to_level", &Ciphertext::drop_to_level)
        .def("add_inplace", &Ciphertext::add_inplace)
        .def("sub_inplace", &Ciphertext::sub_inplace);

    py::class_<SwitchingKey>(m, "SwitchingKey")
        .def_readonly("b", &SwitchingKey::b)
        .def_readonly("a", &SwitchingKey::a)
        .def_readonly("from_id", &SwitchingKey::from_id)
        .def_readonly("to_id", &SwitchingKey::to_id)
        .def_readonly("a_seed", &SwitchingKey::a_seed);

    py::class_<EvalKeys>(m, "EvalKeys")
        .def(py::init<>())
        .def_readwrite("relin", &EvalKeys::relin)
        .def("add_galois", [](EvalKeys& k, u64 g, const SwitchingKey& s) { k.galois[g] = s; })
        .def("has", &EvalKeys::has)
        .def("galois_exponents", [](const EvalKeys& k) {
            std::vector<u64> v;
            for (auto& [g, s] : k.galois) v.push_back(g);
            return v;
        })
        .def("galois_key", &EvalKeys::galois_key, py::return_value_policy::reference_internal);

    py::class_<KeyContext>(m, "KeyContext")
        .def(py::init<const RingParams&, NoiseParams, GadgetVector>(), py::keep_alive<1, 2>())
        .def("keygen", &KeyContext::keygen)
        .def("relin_key_gen", &KeyContext::relin_key_gen)
        .def("galois_key_gen", &KeyContext::galois_key_gen)
        .def("switch_key_gen", &KeyContext::switch_key_gen)
        .def("encrypt", &KeyContext::encrypt, py::arg("sk"), py::arg("m"), py::arg("scale"), py::arg("rng"),
             py::arg("domain") = Domain::coeffs)
        .def("encrypt_pk", &KeyContext::encrypt_pk, py::arg("pk"), py::arg("m"), py::arg("scale"),
             py::arg("rng"), py::arg("domain") = Domain::coeffs)
        .def("decrypt", &KeyContext::decrypt)
        .def("zero_ciphertext", &KeyContext::zero_ciphertext, py::arg("level"), py::arg("scale"),
             py::arg("sk_id"), py::arg("domain") = Domain::coeffs)
        .def("decompose", [](const KeyContext& c, const Poly& d) { return c.plan().decompose(d); })
        .def("digit_count", [](const KeyContext& c, int level) { return c.plan().digit_count(level); })
        .def("ks_inner", &KeyContext::ks_inner)
        .def("switch_key_apply", &KeyContext::switch_key_apply)
        .def("mod_down_p", &KeyContext::mod_down_p)
        .def("relinearize", &KeyContext::relinearize)
        .def("apply_galois", &KeyContext::apply_galois)
        .def("square_secret", &KeyContext::square_secret);

    m.def("rotation_exponent", &rotation_exponent);
    m.def("conjugation_exponent", &conjugation_exponent);

    py::class_<Encoder>(m, "Encoder")
        .def(py::init<const RingParams&, u32>(), py::keep_alive<1, 2>())
        .def("slots", &Encoder::slots)
        .def("encode_slots", &Encoder::encode_slots)
        .def("decode_slots", &Encoder::decode_slots)
        .def("encode_coeffs", &Encoder::encode_coeffs)
        .def("decode_coeffs", &Encoder::decode_coeffs)
        // The reference's own Encoder::encode_slots (ckks.hpp:70-86, O(n^2)
        // DFT) on every row of `arr` ([batch][slots] complex128), rows spread
        // over a std::thread pool: the unmodified code, only run concurrently
        // (the encoder is const and shares nothing mutable).
        .def("encode_slots_many",
             [](const Encoder& enc, py::array_t<std::complex<double>, py::array::c_style | py::array::forcecast> arr,
                double scale, int level, int threads) {
                 if (arr.ndim() != 2 || arr.shape(1) != py::ssize_t(enc.slots()))
                     throw TetrisError("oracle", "encode_slots_many: shape mismatch");
                 const size_t B = size_t(arr.shape(0)), n = enc.slots();
                 std::vector<std::vector<cplx>> in(B);
                 for (size_t b = 0; b < B; ++b) in[b].assign(arr.data() + b * n, arr.data() + (b + 1) * n);
                 std::vector<Poly> out(B);
                 {
                     py::gil_scoped_release nogil;
                     std::atomic<size_t> next{0};
                     std::exception_ptr err;
                     std::mutex mu;
                     auto worker = [&]() {
                         for (size_t b; (b = next.fetch_add(1)) < B;) {
                             try {
                                 out[b] = enc.encode_slots(in[b], scale, level);
                             } catch (...) {
                                 std::lock_guard<std::mutex> g(mu);
                                 err = std::current_exception();
                             }
                         }
                     };
                     std::vector<std::thread> pool;
                     const int nt = std::max(1, std::min<int>(threads, int(B)));
                     for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
                     for (auto& th : pool) th.join();
                     if (err) std::rethrow_exception(err);
                 }
                 return out;
             },
             py::arg("arr"), py::arg("scale"), py::arg("level"), py::arg("threads") = 1);

    py::class_<Evaluator>(m, "Evaluator")
        .def(py::init<const KeyContext&>(), py::keep_alive<1, 2>())
        .def("ring", &Evaluator::ring, py::return_value_policy::reference_internal)
        .def("key_context", &Evaluator::key_context, py::return_value_policy::reference_internal)
        .def("add", &Evaluator::add, py::call_guard<py::gil_scoped_release>())
        .def("sub", &Evaluator::sub, py::call_guard<py::gil_scoped_release>())
        .def("mul", &Evaluator::mul, py::call_guard<py::gil_scoped_release>())
        .def("mul_relin", &Evaluator::mul_relin, py::call_guard<py::gil_scoped_release>())
        .def("mul_plain", &Evaluator::mul_plain, py::call_guard<py::gil_scoped_release>())
        .def("mul_scalar", &Evaluator::mul_scalar, py::call_guard<py::gil_scoped_release>())
        .def("add_scalar", &Evaluator::add_scalar, py::call_guard<py::gil_scoped_release>())
        .def("rescale", &Evaluator::rescale, py::call_guard<py::gil_scoped_release>())
        .def("rotate", &Evaluator::rotate, py::call_guard<py::gil_scoped_release>())
        .def("conjugate", &Evaluator::conjugate, py::call_guard<py::gil_scoped_release>())
        .def("apply_galois_many", &Evaluator::apply_galois_many, py::call_guard<py::gil_scoped_release>())
        .def_static("scaled_residue", &Evaluator::scaled_residue);

    py::class_<LinearTransformPlan>(m, "LinearTransformPlan")
        .def(py::init<const Encoder&, const std::map<u32, std::vector<cplx>>&, double, int>(), py::keep_alive<1, 2>())
        .def_static("diagonals_of", &LinearTransformPlan::diagonals_of)
        .def("required_rotations", &LinearTransformPlan::required_rotations)
        .def("plain_scale", &LinearTransformPlan::plain_scale)
        .def("baby_count", &LinearTransformPlan::baby_count)
        .def("apply", &LinearTransformPlan::apply, py::call_guard<py::gil_scoped_release>());

    m.def("eval_chebyshev", &eval_chebyshev, py::call_guard<py::gil_scoped_release>());
    m.def("inner_sum", &inner_sum, py::call_guard<py::gil_scoped_release>());
    m.def("power_to_chebyshev", &power_to_chebyshev);

    py::class_<ThresholdParams>(m, "ThresholdParams")
        .def(py::init([](u32 alpha, u32 beta, std::vector<u32> degrees, double eps) {
                 return ThresholdParams{alpha, beta, std::move(degrees), eps};
             }),
             py::arg("alpha") = 8, py::arg("beta") = 12, py::arg("degrees") = std::vector<u32>{},
             py::arg("epsilon") = 1.0)
        .def_readwrite("alpha", &ThresholdParams::alpha)
        .def_readwrite("beta", &ThresholdParams::beta)
        .def_readwrite("degrees", &ThresholdParams::degrees)
        .def_readwrite("epsilon", &ThresholdParams::epsilon);
    py::class_<ChainStage>(m, "ChainStage")
        .def(py::init<>())
        .def_readwrite("degree", &ChainStage::degree)
        .def_readwrite("gamma", &ChainStage::gamma)
        .def_readwrite("upper", &ChainStage::upper)
        .def_readwrite("cheb", &ChainStage::cheb)
        .def_readwrite("error", &ChainStage::error);
    py::class_<MinimaxChain>(m, "MinimaxChain")
        .def(py::init<>())
        .def_readwrite("params", &MinimaxChain::params)
        .def_readwrite("stages", &MinimaxChain::stages)
        .def_readwrite("sign_error", &MinimaxChain::sign_error)
        .def_readwrite("achieved_beta", &MinimaxChain::achieved_beta)
        .def("eval_coeffs", &MinimaxChain::eval_coeffs)
        .def("eval_step", &MinimaxChain::eval_step)
        .def("levels_required", &MinimaxChain::levels_required);
    m.def("build_chain", &build_chain, py::call_guard<py::gil_scoped_release>());
    m.def("eval_private_threshold", &eval_private_threshold, py::call_guard<py::gil_scoped_release>());
    m.def("eval_private_threshold_plain_norm", &eval_private_threshold_plain_norm, py::call_guard<py::gil_scoped_release>());


    // ---- Half-BTS (bootstrap.hpp) ----
    py::class_<EvalModConfig>(m, "EvalModConfig")
        .def(py::init([](u32 d, u32 a, u32 k, u32 s, double w) { return EvalModConfig{d, a, k, s, w}; }),
             py::arg("cheb_degree") = 30, py::arg("double_angles") = 3, py::arg("lattice_bound") = 16,
             py::arg("arcsine_degree") = 7, py::arg("arcsine_window") = 0.65)
        .def_readwrite("cheb_degree", &EvalModConfig::cheb_degree)
        .def_readwrite("double_angles", &EvalModConfig::double_angles)
        .def_readwrite("lattice_bound", &EvalModConfig::lattice_bound)
        .def_readwrite("arcsine_degree", &EvalModConfig::arcsine_degree)
        .def_readwrite("arcsine_window", &EvalModConfig::arcsine_window);
    py::class_<BootstrapParams>(m, "BootstrapParams")
        .def(py::init<>())
        .def_readwrite("slots", &BootstrapParams::slots)
        .def_readwrite("sparse_log_gap", &BootstrapParams::sparse_log_gap)
        .def_readwrite("secret_hw", &BootstrapParams::secret_hw)
        .def_readwrite("ephemeral_hw", &BootstrapParams::ephemeral_hw)
        .def_readwrite("evalmod", &BootstrapParams::evalmod)
        .def_readwrite("delta_input", &BootstrapParams::delta_input)
        .def_readwrite("delta_evalmod", &BootstrapParams::delta_evalmod)
        .def("depth", &BootstrapParams::depth);
    py::class_<BootstrapEvaluator>(m, "BootstrapEvaluator")
        .def(py::init<const KeyContext&, BootstrapParams>(), py::keep_alive<1, 2>(),
             py::call_guard<py::gil_scoped_release>())
        .def("required_galois_exponents", &BootstrapEvaluator::required_galois_exponents)
        .def("trace_exponents", &BootstrapEvaluator::trace_exponents)
        .def("output_level", &BootstrapEvaluator::output_level)
        .def("mod_raise", &BootstrapEvaluator::mod_raise, py::call_guard<py::gil_scoped_release>())
        .def("trace_map", &BootstrapEvaluator::trace_map, py::call_guard<py::gil_scoped_release>())
        .def("coeffs_to_slots", &BootstrapEvaluator::coeffs_to_slots, py::call_guard<py::gil_scoped_release>())
        .def("eval_mod", &BootstrapEvaluator::eval_mod, py::call_guard<py::gil_scoped_release>())
        .def("slots_to_coeffs", &BootstrapEvaluator::slots_to_coeffs, py::call_guard<py::gil_scoped_release>())
        .def("half_bts", &BootstrapEvaluator::half_bts, py::call_guard<py::gil_scoped_release>());

    // ---- wire formats (serialize.hpp) ----
    auto to_bytes = [](const std::vector<uint8_t>& v) { return py::bytes(reinterpret_cast<const char*>(v.data()), v.size()); };
    auto from_bytes = [](const py::bytes& b) {
        std::string s = b;
        return std::vector<uint8_t>(s.begin(), s.end());
    };
    m.def("serialize_ciphertext", [to_bytes](const Ciphertext& c) { return to_bytes(serialize_ciphertext(c)); });
    m.def("deserialize_ciphertext", [from_bytes](const py::bytes& b, const RingParams& r) {
        return deserialize_ciphertext(from_bytes(b), r); });
    m.def("ciphertext_size", &ciphertext_size, py::arg("ring"), py::arg("level"), py::arg("parts") = 2);
    m.def("serialize_switching_key", [to_bytes](const SwitchingKey& k) { return to_bytes(serialize_switching_key(k)); });
    m.def("deserialize_switching_key", [from_bytes](const py::bytes& b, const RingParams& r) {
        return deserialize_switching_key(from_bytes(b), r); });
    m.def("serialize_chain", [to_bytes](const MinimaxChain& c) { return to_bytes(serialize_chain(c)); });
    m.def("deserialize_chain", [from_bytes](const py::bytes& b) { return deserialize_chain(from_bytes(b)); });
    m.def("serialize_secret_key", [to_bytes](const SecretKey& k) { return to_bytes(serialize_secret_key(k)); });
    m.def("deserialize_secret_key", [from_bytes](const py::bytes& b, const RingParams& r) {
        return deserialize_secret_key(from_bytes(b), r); });

    // ---- PFE, repacking, ring merge/split (pfe.hpp, repack.hpp, rlwe.hpp:684-802) ----
    auto ct_ptrs = [](const py::list& l) {
        std::vector<const Ciphertext*> v;
        for (auto h : l) v.push_back(h.is_none() ? nullptr : &h.cast<const Ciphertext&>());
        return v;
    };
    py::class_<FunctionSpec>(m, "FunctionSpec")
        .def(py::init<>())
        .def_readwrite("lo", &FunctionSpec::lo)
        .def_readwrite("hi", &FunctionSpec::hi)
        .def_readwrite("table", &FunctionSpec::table)
        .def_readwrite("out_min", &FunctionSpec::out_min)
        .def_readwrite("out_max", &FunctionSpec::out_max)
        .def("max_value", &FunctionSpec::max_value)
        .def("validate", &FunctionSpec::validate);
    py::class_<TestVector>(m, "TestVector")
        .def(py::init<>())
        .def_readwrite("ct", &TestVector::ct)
        .def_readwrite("lo", &TestVector::lo)
        .def_readwrite("hi", &TestVector::hi)
        .def_readwrite("max_value", &TestVector::max_value);
    m.def("encode_input", &encode_input);
    m.def("build_test_vector", &build_test_vector);
    m.def("lookup", &lookup);
    m.def("eval_scores", [](const std::vector<std::vector<double>>& rows, const std::vector<TestVector>& tvs,
                            bool trace) {
        std::vector<std::string> t;
        auto out = eval_scores(rows, tvs, trace ? &t : nullptr);
        return py::make_tuple(out, t);
    }, py::arg("rows"), py::arg("tvs"), py::arg("trace") = false);
    py::class_<RepackKeySet>(m, "RepackKeySet")
        .def(py::init<>())
        .def_readwrite("exponents", &RepackKeySet::exponents)
        .def_readwrite("keys", &RepackKeySet::keys)
        .def_readwrite("sk_id", &RepackKeySet::sk_id);
    m.def("repack_exponents", &repack_exponents);
    m.def("gen_repack_keys", &gen_repack_keys);
    m.def("repack", [ct_ptrs](const KeyContext& ctx, const py::list& cts, const RepackKeySet& keys) {
        RepackStats st;
        auto v = ct_ptrs(cts);
        Ciphertext out;
        {
            py::gil_scoped_release nogil;
            out = repack(ctx, v, keys, &st);
        }
        return py::make_tuple(out, st.automorphisms);
    });
    m.def("embed_secret", &embed_secret);
    m.def("merge_embed", [ct_ptrs](const py::list& cts, const RingParams& big) { return merge_embed(ct_ptrs(cts), big); });
    m.def("ring_merge", &ring_merge);
    m.def("ring_merge_many", [ct_ptrs](const KeyContext& ctx, const py::list& cts, const SwitchingKey& swk) {
        return ring_merge_many(ctx, ct_ptrs(cts), swk);
    });
    m.def("ring_split", &ring_split);
    // ---- the exploration protocol (profile.hpp, protocol.hpp) ----
    py::class_<Profile>(m, "Profile")
        .def_static("toy_small", &Profile::toy_small)
        .def_static("toy", &Profile::toy)
        .def_readwrite("n_small", &Profile::n_small)
        .def_readwrite("n_big", &Profile::n_big)
        .def_readwrite("th_local", &Profile::th_local)
        .def_readwrite("th_global", &Profile::th_global)
        .def_readwrite("hw_big", &Profile::hw_big)
        .def_readwrite("evalmod", &Profile::evalmod)
        .def_readwrite("delta_tv", &Profile::delta_tv)
        .def_readwrite("delta_evalmod", &Profile::delta_evalmod)
        .def_readwrite("gadget_group", &Profile::gadget_group)
        .def_readwrite("special_count", &Profile::special_count);
    py::class_<ProtocolContext>(m, "ProtocolContext")
        .def(py::init<Profile>(), py::call_guard<py::gil_scoped_release>())
        .def("ring_small", &ProtocolContext::ring_small, py::return_value_policy::reference_internal)
        .def("ring_big", &ProtocolContext::ring_big, py::return_value_policy::reference_internal)
        .def("ctx_small", &ProtocolContext::ctx_small, py::return_value_policy::reference_internal)
        .def("ctx_big", &ProtocolContext::ctx_big, py::return_value_policy::reference_internal)
        .def("evaluator", &ProtocolContext::evaluator, py::return_value_policy::reference_internal)
        .def("bts", &ProtocolContext::bts, py::return_value_policy::reference_internal)
        .def("chain_local", &ProtocolContext::chain_local, py::return_value_policy::reference_internal)
        .def("chain_global", &ProtocolContext::chain_global, py::return_value_policy::reference_internal)
        .def("galois_manifest", &ProtocolContext::galois_manifest)
        .def("profile", &ProtocolContext::profile, py::return_value_policy::reference_internal);
    py::class_<Query>(m, "Query")
        .def_readonly("t0", &Query::t0)
        .def_readonly("t1", &Query::t1)
        .def_readonly("norm", &Query::norm)
        .def_readonly("small_sk_id", &Query::small_sk_id)
        .def_readonly("big_sk_id", &Query::big_sk_id);
    py::class_<EvalKeySet>(m, "EvalKeySet")
        .def_readonly("merge", &EvalKeySet::merge)
        .def_readonly("big", &EvalKeySet::big, py::return_value_policy::reference_internal)
        .def_readonly("repack", &EvalKeySet::repack);
    py::class_<ScientistSetup>(m, "ScientistSetup")
        .def_readonly("sk_small", &ScientistSetup::sk_small)
        .def_readonly("sk_big", &ScientistSetup::sk_big)
        .def_readonly("keys", &ScientistSetup::keys, py::return_value_policy::reference_internal)
        .def_readonly("query", &ScientistSetup::query, py::return_value_policy::reference_internal);
    py::class_<Database>(m, "Database")
        .def(py::init<>())
        .def_readwrite("attribute_names", &Database::attribute_names)
        .def_readwrite("rows", &Database::rows);
    py::class_<SelectionMatrix>(m, "SelectionMatrix")
        .def_static("identity", &SelectionMatrix::identity);
    m.def("scientist_setup", &scientist_setup, py::call_guard<py::gil_scoped_release>());
    m.def("score_and_repack", &score_and_repack, py::arg("pc"), py::arg("db"), py::arg("sel"), py::arg("query"),
          py::arg("keys"), py::arg("threads") = 1, py::call_guard<py::gil_scoped_release>());
    m.def("explore_from_repacked",
          [](const ProtocolContext& pc, const std::vector<Ciphertext>& repacked, std::size_t p_total,
             const Query& query, const EvalKeySet& keys, int threads) {
              py::gil_scoped_release nogil;
              return explore_from_repacked(pc, repacked, p_total, query, keys, threads);
          },
          py::arg("pc"), py::arg("repacked"), py::arg("p_total"), py::arg("query"), py::arg("keys"),
          py::arg("threads") = 1);

    // Multi-threaded driver for the CPU baseline: evaluates the threshold on
    // each ciphertext with a std::thread pool (the reference's own granularity,
    // protocol.hpp:297-311), sums the outputs in index order and runs
    // inner_sum once (protocol.hpp:319-323). Returns (result, seconds).
    m.def("threshold_count_pool",
          [](const Evaluator& ev, const std::vector<Ciphertext>& scores, const Ciphertext& ct_t, double norm,
             const MinimaxChain& chain, const EvalKeys& keys, u32 slots, int threads, bool do_inner_sum) {
              py::gil_scoped_release nogil;
              auto t0 = std::chrono::steady_clock::now();
              std::vector<Ciphertext> outs(scores.size());
              std::atomic<size_t> next{0};
              std::exception_ptr err;
              std::mutex mu;
              auto worker = [&]() {
                  for (;;) {
                      size_t i = next.fetch_add(1);
                      if (i >= scores.size()) return;
                      try {
                          outs[i] = eval_private_threshold_plain_norm(ev, scores[i], ct_t, norm, chain, keys);
                      } catch (...) {
                          std::lock_guard<std::mutex> g(mu);
                          err = std::current_exception();
                      }
                  }
              };
              std::vector<std::thread> pool;
              int nt = std::max(1, std::min<int>(threads, int(scores.size())));
              for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
              for (auto& th : pool) th.join();
              if (err) std::rethrow_exception(err);
              Ciphertext acc = outs[0];
              for (size_t i = 1; i < outs.size(); ++i) acc = ev.add(acc, outs[i]);
              if (do_inner_sum) acc = inner_sum(ev, acc, slots, keys);
              double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
              return std::make_pair(acc, s);
          });
}
