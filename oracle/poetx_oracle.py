"""CPU oracle for the POET-X hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(`/root/reference/pkg/src/poetx`, "the reference" below).  It exists so
that the CUDA path in ``paper_2603_05500_b200`` can be checked on the GPU
box, where the reference itself is not available.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it, and only as the checker or the
timed CPU baseline -- never as a product code path.

Parity pinning: every function here is checked against golden vectors
produced by running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``).  Because the
restatement keeps the reference's fixed ascending-k rank-1 accumulation
order (``linalg.py:42-60``), the comparison is *bitwise* for float32 and
float64 (see ``tests/test_oracle_golden.py``).

Permutation sampling follows numpy's ``Generator(Philox)`` exactly
(the reference draws permutations through numpy, ``linalg.py:264-291``);
``philox_permutation_py`` is an independent pure-Python restatement of
numpy 2.x's Philox4x64-10 + buffered-uint32 + masked-rejection
Fisher-Yates, pinned against numpy itself.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

# ---------------------------------------------------------------------------
# ordered-accumulation products (reference linalg.py:42-137)
# ---------------------------------------------------------------------------


# Large-shape float64 parity checks (Llama-1B layer shapes, tests/
# test_gpu_bench_config.py) may switch the three dense products to numpy's
# BLAS: in float64 the accumulation order moves results by ~1e-13, far below
# the 2e-2 bf16 tolerance they are checked at, and the ordered loops would
# take minutes per layer.  Every golden/bitwise check keeps the default.
_BLAS = [False]


class blas_products:
    """Context manager: ``with blas_products(): ...`` (float64 only)."""

    def __enter__(self):
        self._old = _BLAS[0]
        _BLAS[0] = True

    def __exit__(self, *exc):
        _BLAS[0] = self._old


def matmul(a, b):
    """a @ b, ascending-k rank-1 accumulation (linalg.py:42-60)."""
    if _BLAS[0] and a.dtype == np.float64:
        return np.matmul(a, b)
    m, k = a.shape
    out = np.zeros((m, b.shape[1]), dtype=a.dtype)
    tmp = np.empty_like(out)
    for i in range(k):
        np.multiply(a[:, i, None], b[i, None, :], out=tmp)
        np.add(out, tmp, out=out)
    return out


def matmul_abt(a, b):
    """a @ b.T without the transposed copy (linalg.py:63-83)."""
    if _BLAS[0] and a.dtype == np.float64:
        return np.matmul(a, b.T)
    out = np.zeros((a.shape[0], b.shape[0]), dtype=a.dtype)
    tmp = np.empty_like(out)
    for i in range(a.shape[1]):
        np.multiply(a[:, i, None], b[None, :, i], out=tmp)
        np.add(out, tmp, out=out)
    return out


def batched_matmul(a, b):
    """out[s] = a[s] @ b[s], ascending shared index (linalg.py:110-130)."""
    if _BLAS[0] and a.dtype == np.float64:
        return np.matmul(a, b)
    nb, m, k = a.shape
    out = np.zeros((nb, m, b.shape[2]), dtype=a.dtype)
    tmp = np.empty_like(out)
    for i in range(k):
        np.multiply(a[:, :, i, None], b[:, i, None, :], out=tmp)
        np.add(out, tmp, out=out)
    return out


def bt(a):
    """Per-slice transpose copy (linalg.py:133-137)."""
    return np.ascontiguousarray(a.transpose(0, 2, 1))


def eye_stack(nb, b, dtype):
    out = np.zeros((nb, b, b), dtype=dtype)
    out[:, np.arange(b), np.arange(b)] = 1.0
    return out


# ---------------------------------------------------------------------------
# Cayley-Neumann parameterization (reference cnp.py)
# ---------------------------------------------------------------------------


def num_pairs(b):
    return b * (b - 1) // 2


def skew_from_packed(packed, b):
    """Row-major strict upper triangle -> skew stack (cnp.py:66-78)."""
    nb = packed.shape[0]
    r, c = np.triu_indices(b, k=1)
    q = np.zeros((nb, b, b), dtype=packed.dtype)
    q[:, r, c] = packed
    q[:, c, r] = -packed
    return q


def packed_grad_from_skew_grad(dq):
    """g_(i,j) = dQ_ij - dQ_ji (cnp.py:81-86)."""
    r, c = np.triu_indices(dq.shape[1], k=1)
    return dq[:, r, c] - dq[:, c, r]


def cnp_forward(q, k=3):
    """Truncated Cayley transform; returns (G, Q, Q^2 or powers) (cnp.py:99-125)."""
    if k == 3:
        q2 = batched_matmul(q, q)
        q3 = batched_matmul(q2, q)
        q4 = batched_matmul(q2, q2)
        g = 2.0 * (q + q2 + q3) + q4
        i = np.arange(q.shape[1])
        g[:, i, i] += 1.0
        return g, (q, q2)
    powers = [q]
    for _ in range(k - 1):
        powers.append(batched_matmul(powers[-1], q))
    eye = eye_stack(q.shape[0], q.shape[1], q.dtype)
    series = eye.copy()
    for p in powers:
        series += p
    return batched_matmul(eye + q, series), (q, powers)


def cnp_backward(cache, dg, k=3):
    """Closed-form k=3 adjoint (six products) or generic adjoint (cnp.py:128-158)."""
    q, extra = cache
    if k == 3:
        q2 = extra
        qt, q2t = bt(q), bt(q2)
        n1 = dg
        n2 = batched_matmul(n1, qt) + batched_matmul(qt, n1)
        t3 = batched_matmul(qt, n2)
        t4 = batched_matmul(q2t, n2)
        t5 = batched_matmul(n1, q2t)
        t6 = batched_matmul(n2, q2t)
        return 2.0 * (n1 + n2) + 2.0 * t3 + t4 + 2.0 * t5 + t6
    powers = extra
    eye = eye_stack(q.shape[0], q.shape[1], q.dtype)
    series = eye.copy()
    for p in powers:
        series += p
    tp = [eye] + [bt(p) for p in powers]
    dq = batched_matmul(dg, bt(series))
    ds = batched_matmul(bt(eye + q), dg)
    for i in range(1, k + 1):
        for j in range(i):
            dq = dq + batched_matmul(batched_matmul(tp[j], ds), tp[i - 1 - j])
    return dq


def cayley_exact(q):
    """(I+Q)(I-Q)^{-1} solved in float64 (cnp.py:161-176)."""
    q64 = q.astype(np.float64)
    eye = eye_stack(q.shape[0], q.shape[1], np.float64)
    lhs = np.ascontiguousarray((eye - q64).transpose(0, 2, 1))
    rhs = np.ascontiguousarray((eye + q64).transpose(0, 2, 1))
    sol = np.linalg.solve(lhs, rhs)
    return np.ascontiguousarray(sol.transpose(0, 2, 1)).astype(q.dtype)


# ---------------------------------------------------------------------------
# block-diagonal factors (reference blockdiag.py)
# ---------------------------------------------------------------------------


def apply_to_features(g, x, transpose=False):
    """Segment s of each row maps through block s (or its transpose) (blockdiag.py:58-73)."""
    nb, b, _ = g.shape
    x3 = np.ascontiguousarray(x).reshape(x.shape[0], nb, b)
    if _BLAS[0] and x.dtype == np.float64:
        gg = g.transpose(0, 2, 1) if transpose else g
        return np.einsum("tsk,skj->tsj", x3, gg, optimize=True).reshape(x.shape[0], nb * b)
    out = np.zeros_like(x3)
    tmp = np.empty_like(x3)
    for k in range(b):
        rhs = g[None, :, :, k] if transpose else g[None, :, k, :]
        np.multiply(x3[:, :, k, None], rhs, out=tmp)
        np.add(out, tmp, out=out)
    return out.reshape(x.shape[0], nb * b)


def apply_to_weight_rows(g, w, transpose=False):
    """Left multiply by the factor, segmenting rows (blockdiag.py:76-90)."""
    nb, b, _ = g.shape
    w3 = np.ascontiguousarray(w).reshape(nb, b, w.shape[1])
    if _BLAS[0] and w.dtype == np.float64:
        gg = g.transpose(0, 2, 1) if transpose else g
        return np.matmul(gg, w3).reshape(nb * b, w.shape[1])
    out = np.zeros_like(w3)
    tmp = np.empty_like(w3)
    for k in range(b):
        lhs = g[:, k, :, None] if transpose else g[:, :, k, None]
        np.multiply(lhs, w3[:, k, None, :], out=tmp)
        np.add(out, tmp, out=out)
    return out.reshape(nb * b, w.shape[1])


def segmented_outer(x, y, b):
    """out[s] = sum over tokens (ascending) of x_s^T y_s (blockdiag.py:100-121)."""
    nb = x.shape[1] // b
    x3 = np.ascontiguousarray(x).reshape(x.shape[0], nb, b)
    y3 = np.ascontiguousarray(y).reshape(y.shape[0], nb, b)
    if _BLAS[0] and x.dtype == np.float64:
        return np.einsum("tsi,tsj->sij", x3, y3, optimize=True)
    out = np.zeros((nb, b, b), dtype=x.dtype)
    tmp = np.empty_like(out)
    for a in range(x.shape[0]):
        np.multiply(x3[a, :, :, None], y3[a, :, None, :], out=tmp)
        np.add(out, tmp, out=out)
    return out


def orthogonality_error(g):
    """||G^T G - I||_F over the stack (blockdiag.py:134-138)."""
    gtg = batched_matmul(bt(g), g)
    eye = eye_stack(g.shape[0], g.shape[1], g.dtype)
    return float(np.sqrt(np.sum((gtg - eye) ** 2)))


# ---------------------------------------------------------------------------
# permutations (reference permute.py)
# ---------------------------------------------------------------------------


def svd_singular_values(a, tol=1e-10, max_sweeps=100):
    """One-sided Jacobi singular values, float64, lexicographic pair order and
    the same rotation / stopping rule (linalg.py:166-218).  Returns
    (descending singular values, converged flag, worst residual of the last
    sweep)."""
    w = np.array(a, dtype=np.float64)
    if w.shape[0] < w.shape[1]:
        w = w.T.copy()
    n = w.shape[1]
    if n == 0:
        return np.zeros(0), True, 0.0
    norms = np.einsum("ij,ij->j", w, w)
    worst = 0.0
    for _ in range(max_sweeps):
        rotated = False
        worst = 0.0
        for p in range(n - 1):
            for q in range(p + 1, n):
                alpha, beta = norms[p], norms[q]
                gamma = float(w[:, p] @ w[:, q])
                scale = np.sqrt(alpha * beta)
                if scale <= 0.0 or abs(gamma) <= tol * scale:
                    continue
                worst = max(worst, abs(gamma) / scale)
                rotated = True
                zeta = (beta - alpha) / (2.0 * gamma)
                t = np.copysign(1.0, zeta) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta))
                c = 1.0 / np.sqrt(1.0 + t * t)
                s = c * t
                cp = w[:, p].copy()
                w[:, p] = c * cp - s * w[:, q]
                w[:, q] = s * cp + c * w[:, q]
                norms[p] = float(w[:, p] @ w[:, p])
                norms[q] = float(w[:, q] @ w[:, q])
        if not rotated:
            sv = np.sort(np.sqrt(np.maximum(norms, 0.0)))[::-1].copy()
            return sv, True, 0.0
    sv = np.sort(np.sqrt(np.maximum(norms, 0.0)))[::-1].copy()
    return sv, False, worst


def invert(fwd):
    inv = np.empty_like(fwd)
    inv[fwd] = np.arange(fwd.shape[0], dtype=fwd.dtype)
    return inv


def permute_cols(w, fwd, inv, direction):
    """'forward' = w[:, inv], 'inverse' = w[:, fwd] (permute.py:95-110)."""
    return w[:, inv] if direction == "forward" else w[:, fwd]


def permute_rows(w, fwd, inv, direction):
    """'forward' = w[fwd], 'inverse' = w[inv] (permute.py:86-92)."""
    return w[fwd, :] if direction == "forward" else w[inv, :]


def premerge(w, fwd_in, fwd_out):
    """PM[i,j] = W[pi_in(i), pi_out(j)] (permute.py:113-125, layer.py:161-167)."""
    return np.ascontiguousarray(w[fwd_in, :][:, fwd_out])


# ---------------------------------------------------------------------------
# the layer (reference layer.py:214-314)
# ---------------------------------------------------------------------------


def quantize_rows(w):
    """quant.py:41-48: per-row absmax/127 scale (1.0 for zero rows), codes =
    clip(rint(w / scale), -127, 127) in float64; scales stored in w's dtype."""
    w64 = np.asarray(w).astype(np.float64)
    absmax = np.max(np.abs(w64), axis=1)
    scales = np.where(absmax > 0.0, absmax / 127.0, 1.0)
    codes = np.clip(np.rint(w64 / scales[:, None]), -127, 127).astype(np.int8)
    return codes, scales.astype(np.asarray(w).dtype)


def dequantize_rows(codes, scales):
    """quant.py:50-61: codes in the scales' float type times the row scale."""
    return codes.astype(scales.dtype) * scales[:, None]


class OracleLayer:
    """Holds exactly the reference layer state: base W, packed params, perms.
    ``quantized`` (POET-XQ, mem variant): the base is kept as int8 rows and
    every product reads the dequantized premerged rows (layer.py:188-210 --
    the reference's row/column dequantising loops accumulate in the same
    ascending order as ``matmul``/``matmul_abt`` on the dequantized matrix)."""

    def __init__(self, base, b, fwd_in, fwd_out, k=3, variant="fast", quantized=False):
        self.quantized = quantized
        if quantized:
            self.codes, self.scales = quantize_rows(base)
            base = dequantize_rows(self.codes, self.scales)
        self.base = np.array(base)
        self.b = b
        self.k = k
        self.variant = variant
        self.dtype = self.base.dtype
        self.m, self.n = self.base.shape
        self.q_r = np.zeros((self.m // b, num_pairs(b)), dtype=self.dtype)
        self.q_p = np.zeros((self.n // b, num_pairs(b)), dtype=self.dtype)
        self.merge_count = 0
        self.set_perms(fwd_in, fwd_out)

    def set_perms(self, fwd_in, fwd_out):
        self.fwd_in = np.asarray(fwd_in, dtype=np.int32)
        self.fwd_out = np.asarray(fwd_out, dtype=np.int32)
        self.inv_in = invert(self.fwd_in)
        self.inv_out = invert(self.fwd_out)
        self.pm = premerge(self.base, self.fwd_in, self.fwd_out)

    def factors(self):
        g_r, c_r = cnp_forward(skew_from_packed(self.q_r, self.b), self.k)
        g_p, c_p = cnp_forward(skew_from_packed(self.q_p, self.b), self.k)
        return g_r, c_r, g_p, c_p

    def forward(self, x):
        """layer.py:214-229: gather -> mm1 -> mm2 -> mm3 -> gather."""
        g_r, c_r, g_p, c_p = self.factors()
        u = x[:, self.fwd_in]
        a = apply_to_features(g_r, u)
        t = matmul(a, self.pm)
        v = apply_to_features(g_p, t)
        z = v[:, self.inv_out]
        cache = dict(x=x, g_r=g_r, g_p=g_p, c_r=c_r, c_p=c_p, t=t if self.variant == "fast" else None)
        return z, cache

    def backward(self, cache, dz):
        """layer.py:231-256."""
        dv = dz[:, self.fwd_out]
        t = cache["t"]
        if t is None:
            u = cache["x"][:, self.fwd_in]
            t = matmul(apply_to_features(cache["g_r"], u), self.pm)
        dg_p = segmented_outer(t, dv, self.b)
        dt = apply_to_features(cache["g_p"], dv, transpose=True)
        da = matmul_abt(dt, self.pm)
        u = cache["x"][:, self.fwd_in]
        dg_r = segmented_outer(u, da, self.b)
        du = apply_to_features(cache["g_r"], da, transpose=True)
        dx = du[:, self.inv_in]
        gr = packed_grad_from_skew_grad(cnp_backward(cache["c_r"], dg_r, self.k))
        gp = packed_grad_from_skew_grad(cnp_backward(cache["c_p"], dg_p, self.k))
        return gr, gp, dx

    def transformed_base(self, exact=False):
        """layer.py:260-273: Psi_m^T (G_R PM G_P) Psi_n."""
        q_r = skew_from_packed(self.q_r, self.b)
        q_p = skew_from_packed(self.q_p, self.b)
        if exact:
            g_r, g_p = cayley_exact(q_r), cayley_exact(q_p)
        else:
            g_r, g_p = cnp_forward(q_r, self.k)[0], cnp_forward(q_p, self.k)[0]
        mid = apply_to_weight_rows(g_r, self.pm)
        mid = apply_to_features(g_p, mid)
        return np.ascontiguousarray(mid[self.inv_in, :][:, self.inv_out])

    def merge_and_reinit(self, new_fwd_in, new_fwd_out, exact=False):
        """layer.py:279-314 with the resampled perms passed in explicitly."""
        q_r = skew_from_packed(self.q_r, self.b)
        q_p = skew_from_packed(self.q_p, self.b)
        if exact:
            err_r = orthogonality_error(cayley_exact(q_r))
            err_p = orthogonality_error(cayley_exact(q_p))
        else:
            err_r = orthogonality_error(cnp_forward(q_r, self.k)[0])
            err_p = orthogonality_error(cnp_forward(q_p, self.k)[0])
        self.base = self.transformed_base(exact)
        if self.quantized:  # requantize the transformed base (layer.py:302-303)
            self.codes, self.scales = quantize_rows(self.base)
            self.base = dequantize_rows(self.codes, self.scales)
        self.q_r[...] = 0.0
        self.q_p[...] = 0.0
        self.set_perms(new_fwd_in, new_fwd_out)
        self.merge_count += 1
        return err_r, err_p


# ---------------------------------------------------------------------------
# optimizer step (reference optim.py)
# ---------------------------------------------------------------------------


def lr_at(step, base_lr, total_steps, warmup_steps=0, min_lr_ratio=0.01, poet_lr_scale=0.5, poet=False):
    """optim.py:47-58."""
    scale = poet_lr_scale if poet else 1.0
    if warmup_steps > 0 and step < warmup_steps:
        return scale * base_lr * step / warmup_steps
    floor = min_lr_ratio * base_lr
    progress = min(1.0, (step - warmup_steps) / (total_steps - warmup_steps))
    return scale * (floor + (base_lr - floor) * 0.5 * (1.0 + math.cos(math.pi * progress)))


def clip_threshold_at(step, since, clip_norm=1.0, start=0.01, ramp=10, window=2000):
    """optim.py:61-74."""
    if since is not None and step < window and since < ramp:
        return start + (clip_norm - start) * (since / ramp)
    return clip_norm


def global_clip(grads, threshold):
    """optim.py:77-94 (float64 norm, in-place scale)."""
    norm = math.sqrt(sum(float(np.sum(np.asarray(g, dtype=np.float64) ** 2)) for g in grads.values()))
    if not math.isfinite(norm):
        raise ArithmeticError(f"non-finite gradient norm {norm}")
    if norm > threshold and norm > 0.0:
        f = threshold / norm
        for g in grads.values():
            g *= g.dtype.type(f)
    return norm


def adamw_step(params, grads, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.01):
    """optim.py:127-148, arithmetic in the parameter dtype.  Returns new t."""
    t += 1
    bc1 = 1.0 - beta1**t
    bc2 = 1.0 - beta2**t
    for name, p in params.items():
        g = grads[name]
        if not np.all(np.isfinite(g)):
            raise ArithmeticError(f"non-finite gradient for {name}")
        ty = p.dtype.type
        one = ty(1.0)
        mm, vv = m[name], v[name]
        mm *= ty(beta1)
        mm += (one - ty(beta1)) * g
        vv *= ty(beta2)
        vv += (one - ty(beta2)) * g * g
        mhat = mm / ty(bc1)
        vhat = vv / ty(bc2)
        p *= one - ty(lr * wd)
        p -= ty(lr) * mhat / (np.sqrt(vhat) + ty(eps))
    return t


# ---------------------------------------------------------------------------
# keyed Philox RNG (reference linalg.py:264-291) -- numpy algorithm, restated
# ---------------------------------------------------------------------------

M64 = (1 << 64) - 1
PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B


def keyed_stream(*tags):
    """Second key word of Rng.keyed: blake2b-64 of '/'.join(tags), little endian."""
    text = "/".join(str(t) for t in tags)
    return int.from_bytes(hashlib.blake2b(text.encode("utf-8"), digest_size=8).digest(), "little")


def numpy_rng(seed, stream):
    return np.random.Generator(np.random.Philox(key=np.array([seed & M64, stream & M64], dtype=np.uint64)))


def _philox_block(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for _ in range(10):
        p0 = PHILOX_M0 * c[0]
        p1 = PHILOX_M1 * c[2]
        hi0, lo0 = p0 >> 64, p0 & M64
        hi1, lo1 = p1 >> 64, p1 & M64
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + PHILOX_W0) & M64
        k1 = (k1 + PHILOX_W1) & M64
    return c


class PhiloxPy:
    """numpy's Philox4x64-10 bit generator state machine, in pure Python."""

    def __init__(self, seed=None, stream=None, state=None):
        if state is not None:
            s = state["state"]
            self.ctr = [int(x) for x in s["counter"]]
            self.key = [int(x) for x in s["key"]]
            self.buf = [int(x) for x in state["buffer"]]
            self.pos = int(state["buffer_pos"])
            self.has32 = int(state["has_uint32"])
            self.u32 = int(state["uinteger"])
        else:
            self.ctr = [0, 0, 0, 0]
            self.key = [seed & M64, stream & M64]
            self.buf = [0, 0, 0, 0]
            self.pos = 4
            self.has32 = 0
            self.u32 = 0

    def next64(self):
        if self.pos < 4:
            out = self.buf[self.pos]
            self.pos += 1
            return out
        for i in range(4):
            self.ctr[i] = (self.ctr[i] + 1) & M64
            if self.ctr[i] != 0:
                break
        self.buf = _philox_block(self.ctr, self.key)
        self.pos = 1
        return self.buf[0]

    def next32(self):
        if self.has32:
            self.has32 = 0
            return self.u32
        nxt = self.next64()
        self.has32 = 1
        self.u32 = nxt >> 32
        return nxt & 0xFFFFFFFF

    def interval(self, mx):
        if mx == 0:
            return 0
        mask = mx
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        if mx <= 0xFFFFFFFF:
            while True:
                val = self.next32() & mask
                if val <= mx:
                    return val
        while True:
            val = self.next64() & mask
            if val <= mx:
                return val


def philox_permutation_py(gen: PhiloxPy, n):
    """numpy Generator.permutation(n): arange then Fisher-Yates i = n-1..1."""
    arr = list(range(n))
    for i in range(n - 1, 0, -1):
        j = gen.interval(i)
        arr[i], arr[j] = arr[j], arr[i]
    return np.array(arr, dtype=np.int32)


# ---------------------------------------------------------------------------
# BASELINE configs[0] inputs (tests/golden/make_golden.py draws them through the reference)
# ---------------------------------------------------------------------------


def cfg1_inputs(seed=2603, m=512, n=512, b=64, T=1024, dt=np.float32, scale=0.01):
    """Regenerate BASELINE configs[0] inputs exactly as make_golden.py drew them
    through the reference (init_layer draw order: W, then pi_in, then pi_out)."""
    r = numpy_rng(seed, keyed_stream("layer"))
    base = (r.standard_normal((m, n)) * (1.0 / np.sqrt(m))).astype(dt)
    fwd_in = r.permutation(m).astype(np.int32)
    fwd_out = r.permutation(n).astype(np.int32)
    p = numpy_rng(seed, keyed_stream("packed"))
    q_r = (scale * p.standard_normal((m // b, b * (b - 1) // 2))).astype(dt)
    q_p = (scale * p.standard_normal((n // b, b * (b - 1) // 2))).astype(dt)
    dd = numpy_rng(seed, keyed_stream("data"))
    x = dd.standard_normal((T, m)).astype(dt)
    dz = dd.standard_normal((T, n)).astype(dt)
    return base, fwd_in, fwd_out, q_r, q_p, x, dz
