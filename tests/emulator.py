"""CPU emulator of the section kernel's data flow — TEST INFRASTRUCTURE for the section compiler.

It executes the programs sv_compile_circuit returns exactly as paper_2102_02957_b200/csrc/
section.cu does: per CTA tile, per thread, 16 registers per phase, the swizzled shared-memory
offsets and HBM memory bits of every boundary map, and every op type (U2/U1/H1/PERM2/DIAG/
DIAG_CP/DIAGSET).  On the way it asserts the properties the kernel relies on: every shared-memory
mapping is a bijection of the tile, and each CTA stores exactly the addresses it loaded (in-place
safety).  The gate arithmetic here is plain numpy; parity is judged against the oracle.
"""
import numpy as np

# program.h layout (ints)
H_T, H_NOUT, H_NPH, H_PHOFF, H_OPOFF, H_FLAGS = 0, 2, 3, 4, 5, 7
H_TILE, H_STORE_BITS, H_OUT = 8, 24, 40
H_LOAD, H_STORE, H_DIN, H_DOUT = 88, 128, 168, 208
M_TW, M_RW, M_TMB, M_RMB = 0, 16, 20, 36
PHASE_INTS, P_RW, P_OPB, P_OPC, P_TW = 44, 4, 8, 9, 28
OP_INTS = 8
U2, U1, H1, PERM2, DIAG, DIAG_CP, DIAGSET, H1U = 1, 2, 3, 4, 5, 6, 7, 8
KS = np.arange(16)


def _bits(x, b):
    return (x >> b) & 1


def run_section(mem, prog, coefs, n_out, T, flags, aux=None):
    nt = 1 << (T - 4)
    tids = np.arange(nt)
    first = bool(flags & 1) and bool(flags & 2)  # launch_t runs (first direct, last smem) as smem-only
    last = bool(flags & 2)
    out_bits = prog[H_OUT:H_OUT + n_out]
    nph, phoff, opoff = prog[H_NPH], prog[H_PHOFF], prog[H_OPOFF]

    def hbm(M, tile_off):
        base = np.full(nt, tile_off, dtype=np.int64)
        for j in range(T - 4):
            base |= _bits(tids, j).astype(np.int64) << int(prog[M + M_TMB + j])
        ro = np.zeros(16, dtype=np.int64)
        for s in range(4):
            ro |= _bits(KS, s).astype(np.int64) << int(prog[M + M_RMB + s])
        return base[:, None] | ro[None, :]

    def smem(tw, rw):
        x = np.zeros(nt, dtype=np.int64)
        for j in range(T - 4):
            x ^= _bits(tids, j) * int(prog[tw + j])
        xr = np.zeros(16, dtype=np.int64)
        for s in range(4):
            xr ^= _bits(KS, s) * int(prog[rw + s])
        idx = x[:, None] ^ xr[None, :]
        assert len(np.unique(idx)) == 1 << T, "shared-memory mapping is not a bijection"
        return idx

    for b in range(1 << n_out):
        tile_off = 0
        for j, ob in enumerate(out_bits):
            tile_off |= ((b >> j) & 1) << int(ob)
        sm = np.zeros(1 << T, dtype=np.complex128)
        loaded = hbm(H_DIN if first else H_LOAD, tile_off)
        v = mem[loaded].copy()
        if not first:
            sm[smem(H_LOAD + M_TW, H_LOAD + M_RW)] = v
        stored = None
        for ph in range(nph):
            P = phoff + ph * PHASE_INTS
            x = smem(P + P_TW, P + P_RW)
            if not (first and ph == 0):
                v = sm[x].copy()
            ob, oc = prog[P + P_OPB], prog[P + P_OPC]
            for o in range(oc):
                apply_op(v, prog, coefs, opoff + (ob + o) * OP_INTS, tids, tile_off, aux)
            if last and ph == nph - 1:
                stored = hbm(H_DOUT, tile_off)
                mem[stored] = v
            else:
                sm[x] = v
        if not last:
            v = sm[smem(H_STORE + M_TW, H_STORE + M_RW)]
            stored = hbm(H_STORE, tile_off)
            mem[stored] = v
        assert np.array_equal(np.sort(loaded.ravel()), np.sort(stored.ravel())), "CTA stores outside its tile"


def _bitval(code, k, tids, tile_off):
    """(nt, 16) int array of a DIAG operand's bit for every thread / register."""
    if code < 4:
        return np.broadcast_to(_bits(k, code)[None, :], (len(tids), 16))
    if code < 100:
        return np.broadcast_to(_bits(tids, code - 32)[:, None], (len(tids), 16))
    if code < 200:
        return np.full((len(tids), 16), (tile_off >> (code - 100)) & 1)
    return np.full((len(tids), 16), code - 200)


def apply_op(v, prog, coefs, oi, tids, tile_off, aux=None):
    typ, a, b, cb, extra = (int(x) for x in prog[oi:oi + 5])
    if typ == U2:
        m = coefs[cb:cb + 16].reshape(4, 4)
        for q in range(16):
            if (q >> a) & 1 or (q >> b) & 1:
                continue
            idx = [q, q | 1 << a, q | 1 << b, q | 1 << a | 1 << b]
            v[:, idx] = v[:, idx] @ m.T
    elif typ == U1:
        m = coefs[cb:cb + 4].reshape(2, 2)
        for q in range(16):
            if (q >> a) & 1:
                continue
            idx = [q, q | 1 << a]
            v[:, idx] = v[:, idx] @ m.T
    elif typ == H1:
        s = coefs[cb].real
        for q in range(16):
            if (q >> a) & 1:
                continue
            x, y = v[:, q].copy(), v[:, q | 1 << a].copy()
            v[:, q], v[:, q | 1 << a] = s * (x + y), s * (x - y)
    elif typ == H1U:
        for q in range(16):
            if (q >> a) & 1:
                continue
            x, y = v[:, q].copy(), v[:, q | 1 << a].copy()
            v[:, q], v[:, q | 1 << a] = x + y, x - y
    elif typ == PERM2:
        perm = [(extra >> (2 * s)) & 3 for s in range(4)]
        for q in range(16):
            if (q >> a) & 1 or (q >> b) & 1:
                continue
            idx = [q, q | 1 << a, q | 1 << b, q | 1 << a | 1 << b]
            old = v[:, idx].copy()
            for s in range(4):
                v[:, idx[s]] = old[:, perm[s]]
    elif typ == DIAG:
        d = coefs[cb:cb + 4]
        s = _bitval(a, KS, tids, tile_off) + 2 * _bitval(b, KS, tids, tile_off)
        v *= d[s]
    elif typ == DIAG_CP:
        both = (_bitval(a, KS, tids, tile_off) & _bitval(b, KS, tids, tile_off)).astype(bool)
        v[both] *= coefs[cb]
    elif typ == DIAGSET:
        d = a
        flags, aux0 = int(prog[d]) & 1, int(prog[d + 1])
        nthr = len(tids)
        F = []
        for i in range(5):
            f = 1.0 + 0j
            for t in range(int(prog[d + 2 + i]), int(prog[d + 3 + i]), 3):
                O = (int(prog[t]) & 0xffffffff) | ((int(prog[t + 1]) & 0xffffffff) << 32)
                if tile_off & O == O:
                    f *= coefs[int(prog[t + 2])]
            F.append(f * aux[aux0 + i * nthr + tids])
        for t in range(int(prog[d + 8]), int(prog[d + 9]), 5):
            si, J = int(prog[t]), int(prog[t + 1])
            O = (int(prog[t + 2]) & 0xffffffff) | ((int(prog[t + 3]) & 0xffffffff) << 32)
            if tile_off & O == O:
                sel = (tids & J) == J
                F[si][sel] *= coefs[int(prog[t + 4])]
        for k in range(16):
            f = F[0].copy()
            for s_ in range(4):
                if (k >> s_) & 1:
                    f *= F[1 + s_]
            if flags & 1:
                f *= coefs[cb + k]
            v[:, k] *= f
    else:
        raise AssertionError(f"unknown op type {typ}")


def swap_bits(mem, m1, m2):
    """Physical swap of memory bits m1, m2 (the per-gate swap kernel / an exchange)."""
    n = mem.size.bit_length() - 1
    x = np.arange(mem.size, dtype=np.int64)
    y = x ^ (((((x >> m1) ^ (x >> m2)) & 1)) * ((1 << m1) | (1 << m2)))
    mem[:] = mem[y]


def run(steps, prog, coefs, aux, mem, gate_fn=None):
    """Execute every step on the full memory-ordered state `mem` (in place)."""
    for st in steps:
        kind = int(st[0])
        if kind == 1:
            off, cnt, coff, ccnt, T, n_out, flags, aoff, acnt = (int(x) for x in st[1:10])
            run_section(mem, prog[off:off + cnt], coefs[coff:coff + ccnt], n_out, T, flags, aux[aoff:aoff + acnt])
        elif kind in (0, 3):
            swap_bits(mem, int(st[1]), int(st[2]))
        elif kind == 2:
            gate_fn(mem, st)
        else:
            raise AssertionError(kind)


def smem_conflicts(prog, G):
    """Boundary maps / phases of one section whose 2^G-lane groups would hit a 128-byte smem
    wavefront with a repeated 16-byte (fp64, G=3) / 8-byte (fp32, G=4) slot: the low G bits of
    the first G thread words must be linearly independent (the kernel's offsets are XORs of them)."""
    T, nph, phoff = int(prog[H_T]), int(prog[H_NPH]), int(prog[H_PHOFF])
    ntl = T - 4
    mask = (1 << G) - 1
    bad = []

    def indep(words):
        span = {0}
        for w in words:
            v = w & mask
            if v in span:
                return False
            span |= {u ^ v for u in span}
        return True

    maps = [("load", H_LOAD + M_TW), ("store", H_STORE + M_TW)] + \
           [(f"phase{k}", phoff + k * PHASE_INTS + P_TW) for k in range(nph)]
    for name, tw in maps:
        words = [int(prog[tw + j]) for j in range(min(G, ntl))]
        if ntl >= G and not indep(words):
            bad.append(name)
    return bad
