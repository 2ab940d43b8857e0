"""Shared-memory bank-conflict model of the Stockham exchanges in csrc/fft_core.cuh.

Enumerates every exchange store/load of a forward + inverse line transform for
a (L, E, LPC) configuration, maps threads to (line, t) like the column kernels
(line = tid % LPC, t = tid / LPC) or the row kernels (line = tid / TPL), and
counts 16-byte wavefronts per warp instruction (4 phases of 8 threads; a phase
costs the max number of distinct addresses falling on one 16-byte bank group).
Used to pick the padding / line-stride of the exchange buffers.
"""
import itertools
import sys


def line_params(L, E):
    M = 1 << L
    EPT = M if M <= E else E
    TPL = M // EPT
    LE = E.bit_length() - 1
    NST = 0 if L == 0 else (1 if L <= LE else (L + LE - 1) // LE)
    R0 = M if L <= LE else ((1 << (L % LE)) if L % LE else E)
    frad = [R0] + [E] * (NST - 1)
    return M, EPT, TPL, NST, frad


def exchanges(L, E, inv):
    """Yield (kind, list over t of list over instr of element index)."""
    M, EPT, TPL, NST, frad = line_params(L, E)
    rad = list(reversed(frad)) if inv else frad
    ns = [1]
    for s in range(NST - 1):
        ns.append(ns[-1] * rad[s])
    out = []
    for S in range(NST - 1):
        R, NS = rad[S], ns[S]
        G = EPT // R
        wr = []
        for g in range(G):
            for r in range(R):
                wr.append([((t + g * TPL) // NS) * NS * R + ((t + g * TPL) & (NS - 1)) + r * NS for t in range(TPL)])
        R2 = rad[S + 1]
        G2 = EPT // R2
        rd = []
        for g in range(G2):
            for r in range(R2):
                rd.append([(t + g * TPL) + r * (M // R2) for t in range(TPL)])
        out.append(wr)
        out.append(rd)
    return [ins for ex in out for ins in ex]


def cost(L, E, LPC, addr, mapping="col", il=None):
    M, EPT, TPL, NST, frad = line_params(L, E)
    NT = LPC * TPL
    total = ideal = 0
    for inv in (False, True):
        for ins in exchanges(L, E, inv):
            for w0 in range(0, NT, 32):
                for p in range(4):
                    groups = {}
                    for tid in range(w0 + 8 * p, w0 + 8 * p + 8):
                        if mapping == "col":
                            line, t = tid % LPC, tid // LPC
                        elif mapping == "il":  # groups of il lines interleaved over il*TPL threads
                            grp = il * TPL
                            line, t = (tid // grp) * il + tid % il, (tid % grp) // il
                        else:
                            line, t = tid // TPL, tid % TPL
                        a = addr(line, ins[t])
                        groups.setdefault(a % 8, set()).add(a)
                    total += max(len(s) for s in groups.values())
                    ideal += 1
    return total, ideal


def pad_fn(shifts):
    return lambda i: i + sum(i >> s for s in shifts)


if __name__ == "__main__":
    cfgs = [(12, 16, 1), (10, 16, 4), (11, 16, 2), (9, 16, 8), (12, 8, 1), (11, 8, 1), (10, 8, 2)]
    for L, E, LPC in cfgs:
        M = 1 << L
        base = lambda line, i: line * (M + (M >> 3) + 1) + i + (i >> 3)
        b = cost(L, E, LPC, base)
        res = []
        for shifts in [(3,), (3, 6), (3, 7), (3, 6, 9), (4,), (4, 7), (2,), (3, 5), (4, 6)]:
            pf = pad_fn(shifts)
            size = pf(M - 1) + 1
            for extra in range(8):
                stride = size + extra
                c = cost(L, E, LPC, lambda line, i, pf=pf, stride=stride: line * stride + pf(i))
                res.append((c[0], shifts, extra, size))
        res.sort()
        print(f"L={L} E={E} LPC={LPC}: base {b[0]}/{b[1]} = {b[0]/b[1]:.3f}; best:",
              [(r[0] / b[1], r[1], r[2]) for r in res[:4]])
        sys.stdout.flush()
