import sys, dataclasses, math
sys.path.insert(0, '.')
from paper_2412_13269_b200 import tetris as G, workloads as W
spec = dataclasses.replace(W.CONFIGS[5], n_cts=1, records=1 << 15)
S = W.make_context(G, spec)
chain = W.config3_chain(G, spec)
print("levels_required", chain.levels_required(), [st.degree for st in chain.stages])
print("primes", [round(math.log2(q), 6) for q in S.primes[:6]])
d = W.statement_data(spec)
q = W.statement_query_inputs(S, d)
blk = W.statement_block_inputs(S, d, 0)
for mode in (G.PolyEval.ladder, G.PolyEval.bsgs):
    for name, x, t, norm in (("sugar", blk.ct_sugar, q.ct_t[0], 1.0), ("risk", W.linear_score(S, q.ct_w, blk.pt_attr, blk.attr_scale), q.ct_t[2], 0.5)):
        try:
            diff = S.ev.sub(x, t)
            ql = S.ring.modulus(diff.level())
            u = S.ev.rescale(S.ev.mul_scalar(diff, norm, float(ql)))
            for i in range(len(chain.stages)):
                print(f"  {mode} {name} stage {i} in level {u.level()} scale/2^50 {u.scale / 2**50:.12f}")
                f = G.eval_chebyshev_bsgs if mode == G.PolyEval.bsgs else G.eval_chebyshev
                u = f(S.ev, u, chain.eval_coeffs(i), S.keys)
            print(mode, name, "ok level", u.level())
        except Exception as e:
            print(mode, name, "FAILED", e)
