"""Per-bin radiance fields and the distributions sampled from them.

Drop-in for guiding.py of the reference.  The batched path used by the
renderer — ``generate_fields_batch`` + ``GuideTables`` — runs on the device:
one CTA per bin cone-traces the n x n equal-area octahedral grid, blurs,
floors and builds the CDF data in shared memory (csrc/fields.cu).  The
single-field helpers (RadianceField, GuidingDistribution, sample_guided,
ProductHierarchy, ...) are small host utilities with the reference's
semantics for callers that inspect one field (cli --dump-field, tests).

Reference map: guiding.py:17-24 constants, :27-134 single-field API,
:143-223 product hierarchy, :231-251 batched fields, :254-309 tables.
"""

import ctypes as C

import numpy as np

from . import _dev, _lib, core, scene as scene_mod

EPSILON_FLOOR = 1e-2
UPPER_RES = 8

_uc = (np.arange(UPPER_RES) + 0.5) / UPPER_RES
_UG_U, _UG_V = np.meshgrid(_uc, _uc, indexing="xy")
UPPER_DIRS = core.octa_uv_to_dir(_UG_U, _UG_V)  # [row=v, col=u, 3], host numpy (bit-exact)

_upper_dev = None


def upper_dirs_device():
    global _upper_dev
    if _upper_dev is None:
        _upper_dev = _dev.upload(np.ascontiguousarray(UPPER_DIRS, dtype=np.float64))
    return _upper_dev


# ---------------------------------------------------------------------------
# single-field API (host utilities)
# ---------------------------------------------------------------------------

class RadianceField:
    __slots__ = ("values", "resolution", "origin", "jitter_uv")

    def __init__(self, values, origin, jitter_uv=(0.5, 0.5)):
        self.values = np.asarray(values, dtype=np.float64)
        self.resolution = self.values.shape[0]
        self.origin = np.asarray(origin, dtype=np.float64)
        self.jitter_uv = jitter_uv


class GuidingDistribution:
    """Marginal CDF over rows + per-row conditional CDFs; ``pdf_table[j, i]``
    = value * N^2 / (total * 4 pi)."""

    __slots__ = ("field", "marginal_cdf", "conditional_cdf", "pdf_table", "total")

    def __init__(self, field):
        v = field.values
        n = field.resolution
        rows = v.sum(axis=1)
        total = float(rows.sum())
        if total <= 0.0:
            raise ValueError("field has no mass; the epsilon floor should prevent this")
        self.field = field
        self.total = total
        self.marginal_cdf = np.cumsum(rows) / total
        self.conditional_cdf = np.cumsum(v, axis=1) / rows[:, None]
        self.pdf_table = v * (n * n / (total * 4.0 * np.pi))


def select_origin(bin_positions, rng):
    k = min(int(rng.next() * len(bin_positions)), len(bin_positions) - 1)
    return np.asarray(bin_positions[k], dtype=np.float64)


def field_cell_directions(n, jitter_uv):
    ju, jv = jitter_uv
    gu, gv = np.meshgrid((np.arange(n) + ju) / n, (np.arange(n) + jv) / n, indexing="xy")
    return core.octa_uv_to_dir(gu, gv)


def generate_field(svo, scene, origin, n, rng=None, jitter=True, blur_sigma=1.0,
                   epsilon=EPSILON_FLOOR):
    """One n x n field at ``origin`` (cone traced on the device)."""
    if jitter:
        if rng is None:
            raise ValueError("jitter requires an rng stream")
        ju, jv = rng.next(), rng.next()
    else:
        ju = jv = 0.5
    from . import backend_cuda

    dirs = field_cell_directions(n, (ju, jv)).reshape(-1, 3)
    rgb = backend_cuda.trace_cones(svo, scene, origin, dirs, 4.0 * np.pi / (n * n))
    vals = core.luminance(rgb).reshape(n, n)
    if blur_sigma > 0.0:
        vals = core.gaussian_blur(vals, blur_sigma)
    return RadianceField(np.maximum(vals, epsilon), origin, (ju, jv))


def build_distribution(field):
    return GuidingDistribution(field)


def _invert_cdf(cdf, u):
    i = min(int(np.searchsorted(cdf, u, side="right")), len(cdf) - 1)
    lo = cdf[i - 1] if i > 0 else 0.0
    span = cdf[i] - lo
    frac = (u - lo) / span if span > 0 else 0.0
    return i, min(frac, 1.0 - 1e-12)


def sample_guided(dist, u1, u2):
    n = dist.field.resolution
    j, fv = _invert_cdf(dist.marginal_cdf, u1)
    i, fu = _invert_cdf(dist.conditional_cdf[j], u2)
    d = core.octa_uv_to_dir((i + fu) / n, (j + fv) / n)
    return d, pdf_guided(dist, d)


def pdf_guided(dist, direction):
    n = dist.field.resolution
    u, v = core.octa_dir_to_uv(np.asarray(direction, dtype=np.float64))
    return float(dist.pdf_table[min(int(v * n), n - 1), min(int(u * n), n - 1)])


class ProductHierarchy:
    __slots__ = ("field", "upper", "upper_cdf_marg", "upper_cdf_cond", "block", "block_sums",
                 "upper_sum")

    def __init__(self, field, upper):
        m = field.resolution // UPPER_RES
        self.field = field
        self.block = m
        self.block_sums = field.values.reshape(UPPER_RES, m, UPPER_RES, m).sum(axis=(1, 3))
        self.upper = upper
        self.upper_sum = float(upper.sum())
        row = upper.sum(axis=1)
        self.upper_cdf_marg = np.cumsum(row) / row.sum()
        self.upper_cdf_cond = np.cumsum(upper, axis=1) / row[:, None]


def bsdf_product_factor(material, wo, normal, directions):
    if material.kind != scene_mod.LAMBERT:
        raise ValueError("product guiding requires a non-delta material")
    lum = float(core.luminance(material.rgb)) / np.pi
    return lum * np.maximum(np.einsum("...j,j->...", directions, normal), 0.0)


def build_product(field, material, wo, normal, epsilon=EPSILON_FLOOR):
    n = field.resolution
    if n < UPPER_RES:
        raise ValueError("field resolution below the upper-layer resolution")
    m = n // UPPER_RES
    means = field.values.reshape(UPPER_RES, m, UPPER_RES, m).mean(axis=(1, 3))
    factor = bsdf_product_factor(material, wo, np.asarray(normal, dtype=np.float64), UPPER_DIRS)
    return ProductHierarchy(field, np.maximum(means * factor, epsilon))


def sample_product(hier, u1, u2, u3, u4):
    n, m = hier.field.resolution, hier.block
    bj, _ = _invert_cdf(hier.upper_cdf_marg, u1)
    bi, _ = _invert_cdf(hier.upper_cdf_cond[bj], u2)
    block = hier.field.values[bj * m:(bj + 1) * m, bi * m:(bi + 1) * m]
    rows = block.sum(axis=1)
    j, fv = _invert_cdf(np.cumsum(rows) / rows.sum(), u3)
    i, fu = _invert_cdf(np.cumsum(block[j]) / rows[j], u4)
    d = core.octa_uv_to_dir((bi * m + i + fu) / n, (bj * m + j + fv) / n)
    return d, pdf_product(hier, d)


def pdf_product_cell(hier, j, i):
    m, n = hier.block, hier.field.resolution
    bj, bi = j // m, i // m
    p_up = hier.upper[bj, bi] / hier.upper_sum
    p_cell = hier.field.values[j, i] / hier.block_sums[bj, bi]
    return float(p_up * p_cell * (n * n) / (4.0 * np.pi))


def pdf_product(hier, direction):
    n = hier.field.resolution
    u, v = core.octa_dir_to_uv(np.asarray(direction, dtype=np.float64))
    return pdf_product_cell(hier, min(int(v * n), n - 1), min(int(u * n), n - 1))


# ---------------------------------------------------------------------------
# batched device path
# ---------------------------------------------------------------------------

class GuideTables:
    """Per-depth guide tables, resident on the device.

    Device layout (wfpg_guide): floored values (B,n,n), row sums (B,n),
    marginal CDF (B,n), totals (B,) and product block sums (B,8,8); the
    samplers evaluate the conditional CDFs and pdfs on the fly with the same
    arithmetic as the reference's fill_batch.  The reference's full arrays
    (marg, cond, pdftab, vals, block_sums, blk_marg, blk_cond) are
    materialised on attribute access for inspection and parity tests.
    """

    def __init__(self, mode, n, n_bins):
        self.mode = mode
        self.n = n
        self.block = n // UPPER_RES
        self.n_bins = int(n_bins)
        self.upper_dirs = UPPER_DIRS
        self.epsilon = EPSILON_FLOOR
        b = max(self.n_bins, 1)
        self.d_vals = _dev.zeros((b, n, n), np.float64)
        self.d_row_sum = _dev.zeros((b, n), np.float64)
        self.d_marg = _dev.zeros((b, n), np.float64)
        self.d_total = _dev.zeros((b,), np.float64)
        self.d_block_sums = _dev.zeros((b, 8, 8), np.float64) if mode == 2 else None
        self.d_block_rows = (_dev.zeros((b, 8, 8, max(1, n // 8)), np.float64) if mode == 2
                             else None)
        self.d_cum = _dev.zeros((b, n, n), np.float64)
        self._expanded = None
        self._cum_valid = False

    def abi(self):
        g = _lib.Guide()
        g.mode = self.mode
        g.n = self.n
        g.capacity = max(self.n_bins, 1)
        g.eps = self.epsilon
        g.vals = self.d_vals.data_ptr()
        g.row_sum = self.d_row_sum.data_ptr()
        g.marg = self.d_marg.data_ptr()
        g.total = self.d_total.data_ptr()
        g.block_sums = self.d_block_sums.data_ptr() if self.d_block_sums is not None else None
        g.block_rows = self.d_block_rows.data_ptr() if self.d_block_rows is not None else None
        g.n_bins = None
        g.upper_dirs = upper_dirs_device().data_ptr()
        g.cum = self.d_cum.data_ptr() if self._cum_valid else None
        return g

    def fill_batch(self, values):
        """Tables from stacked floored field values (B, n, n) (guiding.py:293-309)."""
        self.d_vals.copy_(_dev.upload(np.asarray(values, dtype=np.float64).reshape(
            self.d_vals.shape)))
        g = self.abi()
        _lib.call("wfpg_guide_fill", C.byref(g), self.n_bins, _dev.stream())
        self._expanded = None

    def fill_slot(self, slot, dist):
        vals = _dev.download(self.d_vals)
        vals[slot] = dist.field.values
        self.fill_batch(vals)

    def _expand(self):
        if self._expanded is None:
            b, n, m = max(self.n_bins, 1), self.n, self.block
            cond = _dev.zeros((b, n, n), np.float64)
            pdftab = _dev.zeros((b, n, n), np.float64)
            bm = _dev.zeros((b, 8, 8, max(m, 1)), np.float64) if self.mode == 2 else None
            bc = _dev.zeros((b, 8, 8, max(m, 1), max(m, 1)), np.float64) if self.mode == 2 else None
            g = self.abi()
            _lib.call("wfpg_guide_expand", C.byref(g), self.n_bins, _lib.ptr(cond),
                      _lib.ptr(pdftab), _lib.ptr(bm), _lib.ptr(bc), _dev.stream())
            k = self.n_bins
            self._expanded = {
                "marg": _dev.download(self.d_marg)[:k], "cond": _dev.download(cond)[:k],
                "pdftab": _dev.download(pdftab)[:k], "vals": _dev.download(self.d_vals)[:k],
                "block_sums": (_dev.download(self.d_block_sums)[:k] if self.mode == 2
                               else np.zeros((0, 8, 8))),
                "blk_marg": _dev.download(bm)[:k] if self.mode == 2 else np.zeros((0, 8, 8, m)),
                "blk_cond": (_dev.download(bc)[:k] if self.mode == 2
                             else np.zeros((0, 8, 8, m, m))),
            }
        return self._expanded

    @property
    def marg(self):
        return self._expand()["marg"]

    @property
    def cond(self):
        return self._expand()["cond"]

    @property
    def pdftab(self):
        return self._expand()["pdftab"]

    @property
    def vals(self):
        return self._expand()["vals"]

    @property
    def block_sums(self):
        return self._expand()["block_sums"]

    @property
    def blk_marg(self):
        return self._expand()["blk_marg"]

    @property
    def blk_cond(self):
        return self._expand()["blk_cond"]


def blur_params(blur_sigma):
    """(radius, taps) exactly as core._blur_kernel computes them with numpy."""
    if blur_sigma <= 0.0:
        return 0, np.zeros(1)
    taps, radius = core._blur_kernel(blur_sigma)
    if radius > 16:
        raise ValueError("blur_sigma too large for the device blur (radius > 16)")
    return radius, np.ascontiguousarray(taps, dtype=np.float64)


def generate_fields_device(svo, scene, origins, jitters, n, blur_sigma=1.0,
                           epsilon=EPSILON_FLOOR, product=False):
    """Device fields + tables for device (B,3) origins / (B,2) jitters."""
    b = int(origins.shape[0])
    tables = GuideTables(2 if product else 1, n, b)
    tables.epsilon = epsilon
    radius, taps = blur_params(blur_sigma)
    tables._cum_valid = True
    g = tables.abi()
    _lib.call("wfpg_generate_fields", C.byref(scene.abi()), C.byref(svo.abi()),
              _lib.ptr(origins), _lib.ptr(jitters), b, None, n, radius,
              taps.ctypes.data_as(C.POINTER(C.c_double)), C.byref(g), _dev.stream())
    return tables


def generate_fields_batch(svo, scene, origins, n, jitters, blur_sigma=1.0,
                          epsilon=EPSILON_FLOOR):
    """One field per origin (B,3) with jitters (B,2); returns values (B,n,n)."""
    origins = np.atleast_2d(np.asarray(origins, dtype=np.float64))
    jitters = np.atleast_2d(np.asarray(jitters, dtype=np.float64))
    if len(origins) == 0:
        return np.zeros((0, n, n))
    tables = generate_fields_device(svo, scene, _dev.upload(origins), _dev.upload(jitters), n,
                                    blur_sigma, epsilon)
    return _dev.download(tables.d_vals)[:len(origins)]
