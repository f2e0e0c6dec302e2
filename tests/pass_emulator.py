"""Test-only numpy interpreter of qsb_run_pass programs.

Executes the int64 word stream produced by paper_2009_01845_b200/fusion.py with the exact
semantics of csrc/pass.cu (tile addressing, layouts, slot/thread tables, pivot factor order),
so the planner and encoder are verified on CPU before any GPU run.
"""

from __future__ import annotations

import struct

import numpy as np

OP_END, OP_LAYOUT, OP_G1, OP_G2, OP_PIVOT, OP_PARITY, OP_TERM, OP_SCALE = range(8)
H_TILEPOS = 16


def _w2d(w):
    return struct.unpack("<d", struct.pack("<q", int(w)))[0]


def _cplx(words, i):
    return complex(_w2d(words[i]), _w2d(words[i + 1]))


def run_program(psi_in: np.ndarray, words: np.ndarray, dtype=np.complex128) -> np.ndarray:
    w = [int(x) for x in words]
    K, NREG, n = w[2], w[3], w[4]
    TB = K - NREG  # thread bits
    A = 1 << NREG
    n_tiles = w[6]
    flags = w[7]
    tile_pos = w[H_TILEPOS:H_TILEPOS + K]
    ext_pos = w[H_TILEPOS + K:H_TILEPOS + K + n - K]
    ext_out = w[H_TILEPOS + n:H_TILEPOS + n + n - K]
    ops0 = H_TILEPOS + n + (n - K)
    out = np.zeros_like(psi_in)
    J = np.arange(1 << K, dtype=np.int64)
    jbits = [(J >> b) & 1 for b in range(K)]
    scatter = np.zeros(1 << K, dtype=np.int64)
    for b in range(K):
        scatter |= jbits[b] << tile_pos[b]
    # pivot slots -> op offsets
    piv_ops = []
    p = ops0
    while w[p] != OP_END:
        if w[p] == OP_PIVOT:
            piv_ops.append(p)
        p += w[p + 1]
    real = np.float64 if dtype == np.complex128 else np.float32

    for c in range(n_tiles):
        base = 0
        obase = 0
        for m in range(n - K):
            if (c >> m) & 1:
                base |= 1 << ext_pos[m]
                obase |= 1 << (ext_out[m] if flags & 1 else ext_pos[m])
        gidx = base | scatter
        v = psi_in[gidx].astype(dtype)
        ep = {}
        for q in piv_ops:
            a = q + 2
            ne = w[a + 4]
            f = 1.0 + 0j
            for k in range(ne):
                bit = w[a + 5 + 3 * k]
                if (base >> bit) & 1:
                    f = f * _cplx(w, a + 6 + 3 * k)
            ep[w[a]] = f
        p = ops0
        lay = None
        while w[p] != OP_END:
            op, ln = w[p], w[p + 1]
            a = p + 2
            if op == OP_LAYOUT:
                R = w[a:a + NREG]
                Tb = w[a + NREG:a + NREG + TB]
                slot = np.zeros_like(J)
                for i, b in enumerate(R):
                    slot |= jbits[b] << i
                tid = np.zeros_like(J)
                for i, b in enumerate(Tb):
                    tid |= jbits[b] << i
                gthr = np.zeros_like(J)
                for i, b in enumerate(Tb):
                    gthr |= jbits[b] << w[a + NREG + TB + A + i]
                reg_ooff = w[a + NREG + TB + A + TB:a + NREG + TB + A + TB + A]
                thr_opos = w[a + NREG + TB + 2 * A + TB:a + NREG + TB + 2 * A + 2 * TB]
                lay = dict(R=R, Tb=Tb, slot=slot, tid=tid, gthr=gthr, reg_ooff=reg_ooff, thr_opos=thr_opos)
            elif op in (OP_G1, OP_G2):
                if op == OP_G1:
                    ib, kind, gmask, gval, rmask, rval = w[a:a + 6]
                    bits = [lay["R"][ib]]
                    mw = w[a + 6:a + 6 + 8]
                    dim = 2
                else:
                    ih, il, kind, gmask, gval, rmask, rval = w[a:a + 7]
                    bits = [lay["R"][ih], lay["R"][il]]
                    mw = w[a + 7:a + 7 + 32]
                    dim = 4
                mat = np.array([_cplx(mw, 2 * k) for k in range(dim * dim)]).reshape(dim, dim)
                if kind == 1:  # G_REAL: the kernel reads only the real parts
                    mat = mat.real.astype(np.complex128)
                mat = mat.astype(dtype)
                sel = np.ones_like(J, dtype=bool)
                for b in bits:
                    sel &= jbits[b] == 0
                cond = (((base | lay["gthr"]) & gmask) == gval) & ((lay["slot"] & rmask) == rval)
                j0 = J[sel & cond]
                if j0.size:
                    offs = []
                    for r in range(dim):
                        o = 0
                        for i, b in enumerate(bits):
                            if (r >> (len(bits) - 1 - i)) & 1:
                                o |= 1 << b
                        offs.append(o)
                    idx = np.array(offs)[:, None] + j0[None, :]
                    v[idx] = mat @ v[idx]
            elif op == OP_PIVOT:
                slotn, ptype, pval, use_rt, ne = w[a:a + 5]
                nb = 1 << (TB - 4)
                ta = w[a + 5 + 3 * ne:a + 5 + 3 * ne + 32]
                tb = w[a + 5 + 3 * ne + 32:a + 5 + 3 * ne + 32 + 2 * nb]
                rt = w[a + 5 + 3 * ne + 32 + 2 * nb:a + 5 + 3 * ne + 32 + 2 * nb + 2 * A]
                if ptype == 0:
                    act = ((lay["slot"] >> pval) & 1) == 1
                else:
                    act = ((base | lay["gthr"]) & pval) != 0
                tid = lay["tid"]
                e = ep[slotn]
                taa = np.array([_cplx(ta, 2 * k) for k in range(16)])
                tba = np.array([_cplx(tb, 2 * k) for k in range(nb)])
                rta = np.array([_cplx(rt, 2 * k) for k in range(A)])
                f = e * (taa[tid & 15] * tba[tid >> 4])
                f = f.astype(dtype)
                if use_rt:
                    f = f * rta[lay["slot"]].astype(dtype)
                v[act] = v[act] * f[act]
            elif op == OP_PARITY:
                s1, nd = w[a], w[a + 1]
                par = np.zeros_like(J)
                for k in range(64):
                    if (s1 >> k) & 1:
                        par += (gidx >> k) & 1
                for q in range(nd):
                    d, msk = w[a + 2 + 2 * q], w[a + 3 + 2 * q]
                    both = gidx & (gidx >> d) & msk
                    par += np.array([bin(int(x)).count("1") for x in both])
                odd = (par & 1) == 1
                v[odd] = -v[odd]
            elif op == OP_TERM:
                mask, val = w[a], w[a + 1]
                ph = np.asarray(_cplx(w, a + 2)).astype(dtype)
                hit = (gidx & mask) == val
                v[hit] = v[hit] * ph
            elif op == OP_SCALE:
                v = v * np.asarray(_cplx(w, a)).astype(dtype)
            p += ln
        # store with the final layout's output offsets
        oidx = np.zeros_like(J)
        for i in range(NREG):
            pass
        slot = lay["slot"]
        tid = lay["tid"]
        reg_ooff = np.array(lay["reg_ooff"], dtype=np.int64)
        thr_o = np.zeros_like(J)
        for i in range(TB):
            thr_o |= ((tid >> i) & 1) << lay["thr_opos"][i]
        oidx = obase | thr_o | reg_ooff[slot]
        out[oidx] = v
    _ = real
    return out
