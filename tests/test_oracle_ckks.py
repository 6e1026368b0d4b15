"""Known-answer tests of the CPU CKKS golden model (oracle/ckks_ref.c).

Residue parity with the reference is unpinned (the reference has no
residues); these KATs pin the model's own conventions
 and its decrypted results against the reference's slots."""
import numpy as np
import pytest

CFG1 = dict(logN=13, qbits=[60, 40, 40, 40, 40], pbits=[60], logscale=40)


@pytest.fixture(scope="module")
def cfg1(oracle):
    ck = oracle.CKKS(CFG1["logN"], CFG1["qbits"], CFG1["pbits"], CFG1["logscale"])
    ck.keygen(7)
    return ck


def brv(x, b):
    return int(format(x, f"0{b}b")[::-1], 2)


def test_primes_and_roots(oracle):
    for logN, qb, pb in [(13, [60, 40, 40, 40, 40], [60]), (15, [60] + [50] * 12, [60, 60]),
                         (16, [60] + [50] * 16, [60, 60, 60]), (14, [50] * 8, [60])]:
        ck = oracle.CKKS(logN, qb, pb, 40)
        N = 1 << logN
        assert len(set(ck.primes)) == len(ck.primes)
        for q, b in zip(ck.primes, qb + pb):
            assert q % (2 * N) == 1 and q < (1 << b) and q > (1 << (b - 1))
            assert oracle.lib().ck_is_prime(q)
        # largest admissible prime first
        q0 = ck.primes[0]
        c = q0 + 2 * N
        while c < (1 << qb[0]):
            assert not oracle.lib().ck_is_prime(c)
            c += 2 * N
        for i, q in enumerate(ck.primes):
            psi = oracle.lib().ck_root(ck.h, i)
            assert pow(psi, N, q) == q - 1 and pow(psi, 2 * N, q) == 1


def test_ntt_is_evaluation_at_odd_powers(cfg1, oracle):
    N, q = cfg1.N, cfg1.primes[1]
    psi = oracle.lib().ck_root(cfg1.h, 1)
    a = np.random.default_rng(1).integers(0, q, N, dtype=np.uint64)
    A = cfg1.ntt(1, a)
    for i in (0, 1, 7, 4095, N - 1):
        pe = pow(psi, 2 * brv(i, 13) + 1, q)
        val, x = 0, 1
        for j in range(N):
            val = (val + int(a[j]) * x) % q
            x = x * pe % q
        assert val == int(A[i])
    assert np.array_equal(cfg1.ntt(1, A, inverse=True), a)


def test_ntt_convolution_theorem(oracle):
    ck = oracle.CKKS(6, [30, 30], [31], 20)
    N, q = 64, ck.primes[0]
    rng = np.random.default_rng(2)
    a = rng.integers(0, q, N).astype(object)
    b = rng.integers(0, q, N).astype(object)
    c = [0] * N  # negacyclic schoolbook product
    for i in range(N):
        for j in range(N):
            if i + j < N:
                c[i + j] = (c[i + j] + a[i] * b[j]) % q
            else:
                c[i + j - N] = (c[i + j - N] - a[i] * b[j]) % q
    A = ck.ntt(0, np.array(a, dtype=np.uint64))
    B = ck.ntt(0, np.array(b, dtype=np.uint64))
    prod = np.array([int(x) * int(y) % q for x, y in zip(A, B)], dtype=np.uint64)
    assert np.array_equal(ck.ntt(0, prod, inverse=True), np.array(c, dtype=np.uint64))


def test_automorphism_commutes_with_ntt(cfg1, oracle):
    import ctypes as C
    N, q = cfg1.N, cfg1.primes[2]
    a = np.random.default_rng(3).integers(0, q, N, dtype=np.uint64)
    for k in (1, 3, -1, 33, 1000):
        g = cfg1.galois(k)
        sa = np.zeros(N, dtype=np.uint64)
        oracle.lib().ck_automorph_coef(cfg1.h, 2, a.ctypes.data_as(oracle.u64p), sa.ctypes.data_as(oracle.u64p), g)
        A = cfg1.ntt(2, a)
        pa = np.zeros(N, dtype=np.uint64)
        oracle.lib().ck_automorph_ntt(cfg1.h, A.ctypes.data_as(oracle.u64p), pa.ctypes.data_as(oracle.u64p), g)
        assert np.array_equal(cfg1.ntt(2, sa), pa)


def test_galois_element_realises_left_rotation(cfg1, oracle):
    """X -> X^(5^k) rotates slots left by k: out[i] = in[(i+k) mod s] (reference emu.cpp:15-20)."""
    N = cfg1.N
    z = np.random.default_rng(4).uniform(-1, 1, N // 2)
    coef = cfg1.encode_coef(z, 2.0 ** 40)
    for k in (1, -1, 5, 1024, N // 2 - 1):
        g = cfg1.galois(k)
        out = np.zeros(N)
        for i in range(N):  # signed coefficient automorphism
            e = (i * g) % (2 * N)
            if e < N:
                out[e] = coef[i]
            else:
                out[e - N] = -coef[i]
        zz = cfg1.decode(out, 2.0 ** 40)
        assert np.abs(zz - np.roll(z, -k)).max() < 1e-9


def test_encode_decode_round_trip(cfg1):
    z = np.random.default_rng(5).uniform(-1, 1, cfg1.N // 2)
    coef = cfg1.encode_coef(z, 2.0 ** 40)
    assert np.abs(cfg1.decode(coef.astype(np.float64), 2.0 ** 40) - z).max() < 1e-9
    # fewer slots than s: the rest are zero (Engine::encode takes any power of two)
    z4 = np.array([1.0, 2.0, 3.0, 4.0])
    out = cfg1.decode(cfg1.encode_coef(z4, 2.0 ** 40).astype(np.float64), 2.0 ** 40)
    assert np.abs(out[:4] - z4).max() < 1e-9 and np.abs(out[4:]).max() < 1e-9


def test_encrypt_decrypt(cfg1):
    z = np.random.default_rng(6).uniform(-1, 1, cfg1.N // 2)
    ct = cfg1.encrypt(cfg1.encode(z, cfg1.scale, 4), 4, 9000)
    assert np.abs(cfg1.decrypt(ct, 4, cfg1.scale) - z).max() < 1e-8
    # a different encryption seed changes every residue row
    ct2 = cfg1.encrypt(cfg1.encode(z, cfg1.scale, 4), 4, 9001)
    assert not np.array_equal(ct[1], ct2[1])


def test_rotations_and_hoisting(cfg1):
    z = np.random.default_rng(7).uniform(-1, 1, cfg1.N // 2)
    ct = cfg1.encrypt(cfg1.encode(z, cfg1.scale, 4), 4, 9000)
    ks = [1, -1, 33, 0, 4096, -4097]
    hs = cfg1.rotate_hoisted(ct, 4, ks)
    for i, k in enumerate(ks):
        assert np.abs(cfg1.decrypt(hs[i], 4, cfg1.scale) - np.roll(z, -k)).max() < 1e-6
    # a single rotation is a hoisted group of one (same residues)
    assert np.array_equal(cfg1.rotate(ct, 4, 33), hs[2])


def test_mul_plain_rescale(cfg1):
    rng = np.random.default_rng(8)
    z, w = rng.uniform(-1, 1, cfg1.N // 2), rng.uniform(-1, 1, cfg1.N // 2)
    ct = cfg1.encrypt(cfg1.encode(z, cfg1.scale, 4), 4, 9000)
    q4 = float(cfg1.primes[4])
    m = cfg1.mul_plain(ct, cfg1.encode(w, q4, 4), 4)
    out = cfg1.rescale(m, 4)
    assert np.abs(cfg1.decrypt(out, 3, cfg1.scale) - z * w).max() < 1e-7
    s = cfg1.add(ct, ct, 4)
    assert np.abs(cfg1.decrypt(s, 4, cfg1.scale) - 2 * z).max() < 1e-8


@pytest.mark.parametrize("plan", [1, 2, 3, 4, 5])
def test_conv_cfg1_decrypts_to_reference(cfg1, oracle, golden, plan):
    """decrypt(conv) vs the reference conv_plan slots, <= 1e-6 (north star)."""
    c, m, k = 4, 32, 3
    img, filt = oracle.make_inputs(c, m, k, c, 1000, 2000, 0)
    ct = cfg1.encrypt(cfg1.encode(img, cfg1.scale, 4), 4, 9000)
    out, sc = cfg1.conv(ct, 4, c, m, k, c, filt, plan)
    assert sc == cfg1.scale
    err = np.abs(cfg1.decrypt(out, 3, sc) - golden["cfg1/slots"]).max()
    assert err < 1e-6, err


@pytest.mark.parametrize("name", ["ms_cfg1_c8", "ms_cfg1_c8to4", "ms_cfg1_c4to8"])
def test_multishard_conv_decrypts_to_reference(cfg1, oracle, golden, name):
    """the golden model's multi-shard conv (fused BSGS over t input / n_out output shards)
    decrypts to the reference's conv_image_shards slots, <= 1e-6."""
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    t = c * m * m // s
    cts = np.stack([cfg1.encrypt(cfg1.encode(img[u * s:(u + 1) * s], cfg1.scale, 4), 4, 9000 + u) for u in range(t)])
    out, sc = cfg1.conv_shards(cts, 4, c, m, k, co, filt)
    dec = np.stack([cfg1.decrypt(out[v], 3, sc) for v in range(out.shape[0])])
    assert np.abs(dec - golden[f"{name}/slots"]).max() < 1e-6


@pytest.mark.parametrize("name", ["cs_cfg1_c2m128", "cs_cfg1_c2to4m128"])
def test_channel_shard_conv_decrypts_to_reference(cfg1, oracle, golden, name):
    """the golden model's channel-shard conv (in-shard + neighbour-spill plaintexts, fused BSGS)
    decrypts to the reference's conv_channel_shards slots, <= 1e-6."""
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    nin = c * m * m // s
    cts = np.stack([cfg1.encrypt(cfg1.encode(img[u * s:(u + 1) * s], cfg1.scale, 4), 4, 9000 + u) for u in range(nin)])
    out, sc = cfg1.conv_channel(cts, 4, c, m, k, co, filt)
    dec = np.stack([cfg1.decrypt(out[v], 3, sc) for v in range(out.shape[0])])
    assert np.abs(dec - golden[f"{name}/slots"]).max() < 1e-6


POOLCONV = ["pc_cfg1_c4m32", "pc_cfg1_c8m32", "pc_cfg1_c16m32", "pc_cfg1_c2m32"]


@pytest.mark.parametrize("name", POOLCONV)
def test_packed_conv_after_pool_decrypts_to_reference(cfg1, oracle, golden, name):
    """the golden model's pooling (downsample_restated over ck_lintrans_src) followed by its
    conv over the pooled packing (ck_conv_packed: tau, rep, duplication) decrypts to the
    reference's convolve(pool(pack(img))) slots."""
    c, m, s, kap, co, si, sf = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, kap, co, si, sf, 0)
    block = m * m
    d_in = s // (block * c) if block * c < s else 1
    chunks = list(np.tile(img, d_in).reshape(-1, s))
    top = 4
    cts = [(cfg1.encrypt(cfg1.encode(x, cfg1.scale, top), top, 9000 + u), top) for u, x in enumerate(chunks)]
    pooled, tau, rep, d, mode = oracle.downsample_restated(oracle.CkksOps(cfg1), cts, c, m, s, True, d_in=d_in)
    lv = pooled[0][1]
    out, sc = cfg1.conv_packed(np.stack([p[0] for p in pooled]), lv, c, m // 2, kap, co, filt, tau, rep, d)
    want = golden[f"{name}/slots"]
    assert out.shape[0] == want.shape[0]
    for u in range(out.shape[0]):
        assert np.abs(cfg1.decrypt(out[u], lv - 1, sc) - want[u]).max() < 1e-6
