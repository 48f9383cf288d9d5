"""CPU port of the reference's two timed algorithms -- TEST / BASELINE INFRASTRUCTURE ONLY.

The reference (pkg/src/convbench/algos.py) is pure Python/NumPy and cannot travel to the
GPU box, so bench.py's reference arm and cpu_baseline time this restatement instead
("kind": "port").  Same loop structure, blocking, float64 accumulation and phase
instrumentation as the reference:

  gemm                        algos.py:142-182  BLIS loops jc -> pc -> ic -> mr x nr tiles,
                                                float64 panels, one fp32 write-back
  conv_baseline_im2col_gemm   algos.py:185-209  one im2col (PRE_REORDER), per (group,
                                                image) gemm into NCHW views
  plan_tiles                  algos.py:254-262  L1/L2-driven tile plan
  conv_main_blocked_direct    algos.py:265-334  per-tile packing from the unpadded input,
                                                f-chunked micro-kernel, NCHW unpack

`ledger` is any object with start(phase)/update(phase) taking the reference Phase
integers (0..6, timing.py:28-35).  Pinned against outputs and phase-call counts of the
reference itself by tests/test_oracle.py (golden fixtures).
"""

from __future__ import annotations

import numpy as np

from .conv_oracle import im2col, output_shape

PRE_ANALYSIS, PRE_REORDER, IN_TILING, IN_PACKING, IN_MICROKERNEL, IN_UNPACKING, POST_REORDER = range(7)
F64 = np.float64


class NullLedger:
    def start(self, phase) -> None:
        pass

    def update(self, phase) -> None:
        pass


def _alloc_out(d, x, b):
    oh, ow = output_shape(d)
    out = np.zeros((d.batch, d.out_channels, oh, ow), dtype=x.dtype)
    if b is not None:
        out[:] = b.reshape(1, -1, 1, 1)
    return out


def _row_panels(blk: np.ndarray, mr: int) -> np.ndarray:
    m, k = blk.shape
    p = np.zeros((-(-m // mr) * mr, k), dtype=F64)
    p[:m] = blk
    return p.reshape(-1, mr, k)


def _col_panels(blk: np.ndarray, nr: int) -> np.ndarray:
    k, n = blk.shape
    p = np.zeros((k, -(-n // nr) * nr), dtype=F64)
    p[:, :n] = blk
    return np.ascontiguousarray(p.reshape(k, -1, nr).swapaxes(0, 1))


def gemm(a, b, c_out, ledger, mc=128, kc=256, nc=512, mr=8, nr=8) -> None:
    """c_out += a @ b with the reference's blocking and per-tile instrumentation."""
    m, k = a.shape
    n = b.shape[1]
    acc = c_out.astype(F64)
    for jc in range(0, n, nc):
        for pc in range(0, k, kc):
            ledger.start(IN_PACKING)
            bp = _col_panels(b[pc:pc + kc, jc:jc + nc], nr)
            ledger.update(IN_PACKING)
            for ic in range(0, m, mc):
                ledger.start(IN_PACKING)
                ap = _row_panels(a[ic:ic + mc, pc:pc + kc], mr)
                ledger.update(IN_PACKING)
                ledger.start(IN_TILING)
                tiles = [(i, j) for j in range(bp.shape[0]) for i in range(ap.shape[0])]
                ledger.update(IN_TILING)
                for i, j in tiles:
                    r0, c0 = ic + i * mr, jc + j * nr
                    rh, cw = min(mr, m - r0), min(nr, n - c0)
                    ledger.start(IN_MICROKERNEL)
                    acc[r0:r0 + rh, c0:c0 + cw] += (ap[i] @ bp[j])[:rh, :cw]
                    ledger.update(IN_MICROKERNEL)
    ledger.start(IN_UNPACKING)
    c_out[:] = acc
    ledger.update(IN_UNPACKING)


def conv_baseline_im2col_gemm(d, x, w, b=None, ledger=None):
    ledger = ledger or NullLedger()
    oh, ow = output_shape(d)
    fpg = d.out_channels // d.groups
    kdim = (d.in_channels // d.groups) * d.k_h * d.k_w
    ledger.start(PRE_REORDER)
    cols = im2col(d, x)
    ledger.update(PRE_REORDER)
    out = _alloc_out(d, x, b)
    wmat = w.reshape(d.out_channels, kdim)
    for g in range(d.groups):
        for n in range(d.batch):
            view = out[n, g * fpg:(g + 1) * fpg].reshape(fpg, oh * ow)
            gemm(wmat[g * fpg:(g + 1) * fpg],
                 cols[g * kdim:(g + 1) * kdim, n * oh * ow:(n + 1) * oh * ow], view, ledger)
    return out


def plan_tiles(d, oh: int, ow: int, l1_bytes: int = 32 * 1024, l2_bytes: int = 1024 * 1024):
    kdim = d.in_channels * d.k_h * d.k_w
    budget = max(1, l2_bytes // (16 * kdim))
    tw = min(ow, max(1, min(budget, 64)))
    th = min(oh, max(1, budget // tw))
    fr = min(d.out_channels, max(8, l1_bytes // (16 * kdim)))
    return th, tw, fr


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


def conv_main_blocked_direct(d, x, w, b=None, ledger=None, l1_bytes=32 * 1024,
                             l2_bytes=1024 * 1024):
    if d.groups != 1 or d.dil_h != 1 or d.dil_w != 1:
        raise ValueError("blocked direct requires groups == 1 and dilation == 1")
    ledger = ledger or NullLedger()
    oh, ow = output_shape(d)
    kh, kw, sh, sw, ph, pw = d.k_h, d.k_w, d.stride_h, d.stride_w, d.pad_h, d.pad_w
    kdim = d.in_channels * kh * kw
    ledger.start(PRE_ANALYSIS)
    th_, tw_, fr = plan_tiles(d, oh, ow, l1_bytes, l2_bytes)
    ledger.update(PRE_ANALYSIS)
    ledger.start(PRE_REORDER)
    wmat = np.ascontiguousarray(w.reshape(d.out_channels, kdim), dtype=F64)
    ledger.update(PRE_REORDER)
    out = _alloc_out(d, x, b)
    for n in range(d.batch):
        for y0 in range(0, oh, th_):
            for x0 in range(0, ow, tw_):
                ledger.start(IN_TILING)
                y1, x1 = min(y0 + th_, oh), min(x0 + tw_, ow)
                th, tw = y1 - y0, x1 - x0
                ledger.update(IN_TILING)
                ledger.start(IN_PACKING)
                patch = np.zeros((d.in_channels, kh, kw, th, tw), dtype=F64)
                for ky in range(kh):
                    lo_y = max(y0, _cdiv(ph - ky, sh))
                    hi_y = min(y1, (d.in_h - 1 + ph - ky) // sh + 1)
                    if lo_y >= hi_y:
                        continue
                    iy = lo_y * sh + ky - ph
                    for kx in range(kw):
                        lo_x = max(x0, _cdiv(pw - kx, sw))
                        hi_x = min(x1, (d.in_w - 1 + pw - kx) // sw + 1)
                        if lo_x >= hi_x:
                            continue
                        ix = lo_x * sw + kx - pw
                        patch[:, ky, kx, lo_y - y0:hi_y - y0, lo_x - x0:hi_x - x0] = \
                            x[n, :, iy:iy + (hi_y - lo_y - 1) * sh + 1:sh,
                              ix:ix + (hi_x - lo_x - 1) * sw + 1:sw]
                pmat = patch.reshape(kdim, th * tw)
                ledger.update(IN_PACKING)
                for f0 in range(0, d.out_channels, fr):
                    f1 = min(f0 + fr, d.out_channels)
                    ledger.start(IN_MICROKERNEL)
                    acc = wmat[f0:f1] @ pmat
                    ledger.update(IN_MICROKERNEL)
                    ledger.start(IN_UNPACKING)
                    out[n, f0:f1, y0:y1, x0:x1] += acc.reshape(f1 - f0, th, tw)
                    ledger.update(IN_UNPACKING)
    return out
