"""Staged host->HBM uploads (bench.py e2e leg): HostUpload.upload_async puts
each group of client ciphertexts on a copy stream behind its own event; after
wait() the views hold exactly the host bytes (same as the synchronous
upload), and a query fed from them gives the same residues."""
import numpy as np
import pytest

from common import assert_ct_equal, enc_slots, make_setup

pytestmark = pytest.mark.gpu


def test_staged_upload_matches_sync(G, gpu_available):
    S = make_setup(G, N=1024, nq=4, K=1, group_size=2, seed=5)
    cts = [enc_slots(S, np.linspace(-1, 1, 32) * (i + 1) / 8, 2.0 ** 40, G.Rng(30 + i)) for i in range(5)]
    metas, off = [], 0
    for c in cts:
        metas.append((off, len(c.parts), c.level(), c.scale, c.sk_id))
        off += len(c.parts) * (c.level() + 1) * 1024
    host = G.pinned_empty([off])
    for c, m in zip(cts, metas):
        G.ciphertext_to_numpy(c, host[m[0]:m[0] + m[1] * (m[2] + 1) * 1024])
    up = G.HostUpload(S.ring, host, metas, G.Form.coeff, G.Domain.slots)
    for step in range(3):
        views = up.upload_async([2, 1, 2])
        up.wait([4])  # the last group: every earlier group has completed too
        for a, b in zip(views, cts):
            assert_ct_equal(a, b, f"staged upload step {step}")
        # a product on the staged views equals the product on the originals
        got = S.ev.mul_relin(views[0], views[3], S.keys)
        assert_ct_equal(got, S.ev.mul_relin(cts[0], cts[3], S.keys), "product on staged views")
    sync = up.upload()
    for a, b in zip(sync, cts):
        assert_ct_equal(a, b, "sync upload")
    with pytest.raises(Exception, match="cover every"):
        up.upload_async([2, 2])
    with pytest.raises(Exception, match="no staged upload"):
        up.wait([7])
