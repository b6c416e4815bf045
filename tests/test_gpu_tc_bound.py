"""Validation of the tensor-core filter bound on the device.

The list scan's fp32 filter distance d^ = |x|^2 + |q|^2 - 2 dot is bounded by
|d^ - delta| <= E with E = e_a |q||x| + e_b (|q|^2 + |x|^2) + e_c; the dot's
share of e_a is alpha (bound_tc1 / bound_tc in scan.cu): the tf32 operand
conversion (analytic: the conversion itself is probed per device) plus an
accumulation term that PTX leaves unspecified and the scan MODELS as
4x round-to-nearest per MMA step (single pass D * 2^-23, split 3 D * 2^-23).

hivf_debug_tc_dot runs the scan's exact MMA sequence (same SWIZZLE_64B
operand layout, same K=8 step order, same split formation) on chosen inputs.
Adversarial inputs aim at the accumulator: products just under one ulp of a
large running sum (lost whole if the adder aligns and truncates each
product), exponent spread, and long cancelling chains at D = 768 (96 k-steps).
The accumulation error is isolated with tf32-exact operands, then the whole
dot (conversion + accumulation, and the split's fp32 combine) is checked
against alpha.  The measured worst ratios go to gpurun_out/tc_bound.json.

Plus a D = 768 parity stress whose neighbour gaps sit inside E, so the scan's
completeness proof fails and the repair / exact paths carry the result.
"""
import json
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

U = 2.0 ** -24
D = 768


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_09138_b200 import Context, lib
    Context(0)  # probes the tensor core's conversion on this device
    return lib()


def tf32(x):
    """Round-to-zero to tf32 (exactly representable operands: no conversion error)."""
    return (np.asarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def tc_dot(L, A, B, split):
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    n = B.shape[0]
    out = np.zeros((128, 2 * n if split == 1 else n), np.float32)
    rc = L.hivf_debug_tc_dot(A.ctypes.data, B.ctypes.data, A.shape[1], n, int(split), out.ctypes.data)
    assert rc == 0, rc
    if split == 1:  # the epilogue's combine: fp32 add of [hi*hi + lo*hi] and [hi*lo]
        return (out[:, :n] + out[:, n:]).astype(np.float32)
    return out


def alpha(split, dim):
    # the dot's share of e_a, as bound_tc / bound_tc1 (scan.cu) state it, without the x1.01 / x1.5 headroom
    if split:
        return 4.0 * 2 ** -20 + 1.5 * dim * 2 ** -22, 1.5 * dim * 2 ** -22
    return 2 ** -9 + 2 ** -20 + 0.5 * dim * 2 ** -22, 0.5 * dim * 2 ** -22


def ratios(L, A, B, split):
    got = tc_dot(L, A, B, split).astype(np.float64)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.linalg.norm(A.astype(np.float64), axis=1)[:, None] * np.linalg.norm(B.astype(np.float64), axis=1)[None, :]
    return np.abs(got - exact) / scale


def adversarial_cases(rng):
    """(name, A[128][D], B[16][D]) with tf32-exact entries."""
    cases = []
    # 1. running sum ~1 after the first k-step, then 760 products of 0.9998 ulp(1)
    #    each (1.4140625^2 * 2^-24): all lost if the adder truncates per product
    a = np.full((128, D), 1.4140625 * 2.0 ** -12, np.float32)
    a[:, 0] = 1.0
    b = np.full((16, D), 1.4140625 * 2.0 ** -12, np.float32)
    b[:, 0] = 1.0
    a[:, 1:8] = 0.0
    cases.append(("sub_ulp_tail", a, b))
    # 2. same, negative tail (sum shrinking toward 1 - eps: truncation direction flips)
    b2 = b.copy()
    b2[:, 8:] *= -1
    cases.append(("sub_ulp_tail_negative", a, b2))
    # 3. per-row varied sub-ulp tails: tail products at 2^-s ulp for s in [0, 4)
    a3 = a.copy()
    for r in range(128):
        a3[r, 8:] = tf32(a3[r, 8:] * np.float32(2.0 ** -(r % 4)) * np.float32(1.0 + (r // 4) / 64.0))
    cases.append(("sub_ulp_tail_mixed", a3, b))
    # 3b. per k-step seven products of 0.9998 ulp and one of 0.4999 ulp: if the
    #     adder keeps quarter-ulp pieces of each product, the kept sum is then
    #     fractional and the final truncation loses up to another half ulp
    a3b = a.copy()
    for s in range(1, D // 8):
        a3b[:, 8 * s + 7] = 1.4140625 * 2.0 ** -13
    cases.append(("sub_ulp_tail_fractional", a3b, b))
    # 3c. tail products of 0.2499 ulp (below a quarter-ulp guard) and of 0.7499 ulp
    for name, sc in (("quarter_ulp_tail", 1.4140625 * 2.0 ** -14), ("three_quarter_ulp_tail", 1.060546875 * 2.0 ** -12)):
        a3c = a.copy()
        a3c[:, 8:] = tf32(np.float32(sc))
        cases.append((name, a3c, b))
    # 4. exponent spread: log-uniform magnitudes over 2^-24..2^0, random signs
    mag = 2.0 ** rng.uniform(-24, 0, (128, D))
    a4 = tf32(mag * rng.choice([-1, 1], (128, D)))
    b4 = tf32(2.0 ** rng.uniform(-24, 0, (16, D)) * rng.choice([-1, 1], (16, D)))
    cases.append(("exponent_spread", a4, b4))
    # 5. cancelling chain: +big / -big pairs inside each k-step, small residue terms
    a5 = tf32(rng.standard_normal((128, D)))
    b5 = np.zeros((16, D), np.float32)
    for j in range(16):
        v = tf32(rng.standard_normal(D))
        v[1::2] = -v[0::2] * a5[0, 0::2] / np.where(a5[0, 1::2] == 0, 1, a5[0, 1::2])
        b5[j] = tf32(v)
    cases.append(("cancelling_pairs", a5, b5))
    # 6. dot ~ 0 by construction: x and q orthogonal up to rounding (max relative error)
    a6 = tf32(rng.standard_normal((128, D)))
    b6 = tf32(rng.standard_normal((16, D)))
    for j in range(16):
        v = b6[j].astype(np.float64)
        v -= a6[j].astype(np.float64) * (a6[j].astype(np.float64) @ v) / (a6[j].astype(np.float64) @ a6[j].astype(np.float64))
        b6[j] = tf32(v)
    cases.append(("near_orthogonal", a6, b6))
    # 7. Gaussian (typical embeddings)
    cases.append(("gaussian", tf32(rng.standard_normal((128, D))), tf32(rng.standard_normal((16, D)))))
    return cases


def test_accumulation_error_inside_model(L):
    import ctypes as C
    rng = np.random.default_rng(7)
    report = {"D": D, "accumulation_only": {}, "full_dot": {}}
    e_a = {}
    for split, kind in ((1, 2), (0, 3)):
        ea, eb, ec = C.c_double(), C.c_double(), C.c_double()
        L.hivf_debug_bound(kind, D, C.byref(ea), C.byref(eb), C.byref(ec))
        e_a[split] = ea.value
    worst_acc = worst_e = 0.0
    for name, A, B in adversarial_cases(rng):
        for split in (0, 1):
            r = ratios(L, A, B, split).max()
            a_full, a_acc = alpha(split, D)
            # the distance d^ = |x|^2 + |q|^2 - 2 dot carries twice the dot's error
            report["accumulation_only"][f"{name}/{'split' if split else 'single'}"] = {
                "max_err_over_xq": float(r), "frac_of_accumulation_model": float(r / a_acc),
                "frac_of_e_a": float(2 * r / e_a[split])}
            worst_acc = max(worst_acc, r / a_acc)
            worst_e = max(worst_e, 2 * r / e_a[split])
            assert r <= a_acc, (name, split, r, a_acc)
    report["worst_frac_of_accumulation_model"] = float(worst_acc)
    report["worst_accumulation_frac_of_e_a"] = float(worst_e)
    # the accumulator's worst adversarial error is under a quarter of the
    # filter bound the scan uses
    assert worst_e <= 0.25, worst_e
    # the model (8 ulp of |x||q| per k-step) keeps >= 2x margin over the worst
    # adversarial accumulation measured on the device
    assert worst_acc <= 0.5, worst_acc
    # full dot: raw fp32 operands (the tensor core converts them), adversarial
    # for the conversion too (mantissas just under a tf32 boundary, same signs)
    full = {
        "gaussian": (rng.standard_normal((128, D)), rng.standard_normal((16, D))),
        "max_truncation": (np.full((128, D), 1.0 + 1023.99 / 1024, np.float32) *
                           rng.choice([1, 2, 4], (128, D)).astype(np.float32),
                           np.full((16, D), 1.0 + 1023.99 / 1024, np.float32)),
        "spread_raw": (2.0 ** rng.uniform(-20, 0, (128, D)) * rng.choice([-1, 1], (128, D)),
                       2.0 ** rng.uniform(-20, 0, (16, D)) * rng.choice([-1, 1], (16, D))),
    }
    for name, (A, B) in full.items():
        A = np.asarray(A, np.float32)
        B = np.asarray(B, np.float32)
        for split in (0, 1):
            r = ratios(L, A, B, split).max()
            a_full, _ = alpha(split, D)
            report["full_dot"][f"{name}/{'split' if split else 'single'}"] = {
                "max_err_over_xq": float(r), "frac_of_alpha": float(r / a_full)}
            assert r <= a_full, (name, split, r, a_full)
    # the coefficients the library actually uses cover alpha with headroom
    for kind, split in ((2, 1), (3, 0)):
        ea, eb, ec = C.c_double(), C.c_double(), C.c_double()
        L.hivf_debug_bound(kind, D, C.byref(ea), C.byref(eb), C.byref(ec))
        assert ea.value >= 2 * alpha(split, D)[0] * 1.4
        report[f"e_a_kind{kind}"] = ea.value
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "tc_bound.json"), "w") as f:
        json.dump(report, f, indent=1)


def f16(x):
    """Round-to-nearest to fp16 (values in the fp16 normal range stay exact afterwards)."""
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)


def alpha_h16(dim):
    # bound_h16 (scan.cu): RN fp16 operands (2^-11 each, Cauchy-Schwarz), the
    # subnormal floor after the per-vector power-of-2 scaling, and the same
    # accumulation allowance as the single-pass tf32 scan (twice the k-steps)
    return 2 ** -10 + 2 ** -22 + 2 * np.sqrt(dim) * 2 ** -38 + 0.5 * dim * 2 ** -22, 0.5 * dim * 2 ** -22


def test_f16_accumulation_error_inside_model(L):
    """The fp16 filter copy's MMA (kind::f16, K = 16 per step, f32 accumulate):
    the same adversarial accumulation cases on fp16-exact operands, then raw
    fp32 operands through the RN conversion, against bound_h16."""
    import ctypes as C
    rng = np.random.default_rng(8)
    report = {"D": D, "accumulation_only": {}, "full_dot": {}}
    ea, eb, ec = C.c_double(), C.c_double(), C.c_double()
    assert L.hivf_debug_bound(4, D, C.byref(ea), C.byref(eb), C.byref(ec)) == 0
    a_full, a_acc = alpha_h16(D)
    assert ea.value >= 2 * a_full * 1.4
    worst = 0.0
    for name, A, B in adversarial_cases(rng):
        if name == "exponent_spread":  # keep inside the fp16 normal range
            A = np.sign(A) * 2.0 ** rng.uniform(-14, 0, A.shape)
            B = np.sign(B) * 2.0 ** rng.uniform(-14, 0, B.shape)
        A, B = f16(A), f16(B)
        r = ratios(L, A, B, 2).max()
        report["accumulation_only"][name] = {"max_err_over_xq": float(r), "frac_of_accumulation_model": float(r / a_acc),
                                             "frac_of_e_a": float(2 * r / ea.value)}
        worst = max(worst, r / a_acc)
        assert r <= a_acc, (name, r, a_acc)
        assert 2 * r / ea.value <= 0.25, name
    assert worst <= 0.5, worst
    report["worst_frac_of_accumulation_model"] = float(worst)
    full = {
        "gaussian": (rng.standard_normal((128, D)) * 900.0, rng.standard_normal((16, D)) * 700.0),
        "max_rounding": (np.full((128, D), 1.0 + 1023.5 / 1024, np.float32) *
                         rng.choice([1, 2, 4], (128, D)).astype(np.float32),
                         np.full((16, D), 1.0 + 1023.5 / 1024, np.float32)),
        "spread_raw": (2.0 ** rng.uniform(-10, 14, (128, D)) * rng.choice([-1, 1], (128, D)),
                       2.0 ** rng.uniform(-10, 14, (16, D)) * rng.choice([-1, 1], (16, D))),
    }
    for name, (A, B) in full.items():
        A = np.asarray(A, np.float32)
        B = np.asarray(B, np.float32)
        r = ratios(L, A, B, 2).max()
        report["full_dot"][name] = {"max_err_over_xq": float(r), "frac_of_alpha": float(r / a_full)}
        assert r <= a_full, (name, r, a_full)
    report["e_a_kind4"] = ea.value
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "tc_bound_f16.json"), "w") as f:
        json.dump(report, f, indent=1)


def test_dim768_parity_with_gaps_inside_the_bound(L):
    """Neighbours on a thin shell around each query: distance gaps ~1e-5
    relative, well inside E, so the scan's completeness proof fails for most
    segments and the repair / exact-fallback paths must produce the
    reference's bits."""
    from paper_2507_09138_b200 import Context, IvfIndex
    rng = np.random.default_rng(11)
    n, K, B = 24000, 24, 40
    Q = rng.standard_normal((B, D)).astype(np.float32)
    rows = []
    for i in range(n):
        q = Q[i % B]
        u = rng.standard_normal(D)
        u /= np.linalg.norm(u)
        rows.append(q + (1.0 + 1e-5 * rng.standard_normal()) * u)
    X = np.asarray(rows, np.float32)
    cents = np.stack([X[rng.choice(n, 200)].mean(0) for _ in range(K)]).astype(np.float32)
    assign = oracle.compute_assignments(X, cents)
    ids = rng.permutation(n).astype(np.uint64)
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign, 0)
    ctx = Context(0)
    for kernel in (3, 2, 1):  # single-pass TC, split TC, FFMA
        ctx.set_option("scan_kernel", kernel)
        try:
            ix = IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids, 0)
            for nprobe, k in ((4, 10), (K, 32)):
                gi, gd, gc = ix.search(Q, nprobe, k)
                oi, od, oc = csr.search(Q, nprobe, k)
                assert np.array_equal(gc, oc)
                assert np.array_equal(gi, oi), kernel
                assert np.array_equal(gd.view(np.uint64), od.view(np.uint64)), kernel
        finally:
            ctx.set_option("scan_kernel", 0)
