import itertools
def patterns(L, E, radices):
    NT = L // E; pats = []
    NS = 1
    for p, R in enumerate(radices):
        NB = E // R
        if p + 1 < len(radices):
            for b in range(NB):
                for r in range(R):
                    acc = []
                    for t in range(NT):
                        j = t + NT * b; k = j % NS; base = (j - k) * R + k
                        acc.append(base + r * NS)
                    pats.append(acc)
            for s in range(E):
                pats.append([t + NT * s for t in range(NT)])
        NS *= R
    return pats
def wavefronts(pats, f, esz):
    per = 128 // esz  # threads per wavefront group (16B: 8, 8B: 16)
    slots = 128 // esz
    tot = ideal = 0
    for acc in pats:
        for w0 in range(0, len(acc), 32):
            warp = acc[w0:w0 + 32]
            for q0 in range(0, len(warp), per):
                grp = warp[q0:q0 + per]
                # wavefronts = max multiplicity of (slot mod slots) distinct rows
                rows = {}
                for e in grp:
                    s = f(e); rows.setdefault(s % slots, set()).add(s // slots)
                tot += max(len(v) for v in rows.values()); ideal += 1
    return tot / ideal
def search(L, E, radices, esz):
    pats = patterns(L, E, radices)
    NT = L // E
    res = []
    cands = {'none': lambda e: e, 'i+i/8': lambda e: e + e // 8, 'i+i/16': lambda e: e + e // 16}
    for P in range(2, 260):
        for Q in (1, 2, 3, 4, 5, 7):
            cands[f'e+e//{P}*{Q}'] = (lambda P, Q: (lambda e: e + (e // P) * Q))(P, Q)
    for name, f in cands.items():
        res.append((wavefronts(pats, f, esz), name))
    res.sort()
    return res[:6], [r for r in res if r[1] in ('none', 'i+i/8', 'i+i/16')]
for (L, E, rad) in [(2000, 20, [20, 20, 5]), (2000, 10, [10, 10, 10, 2]), (512, 8, [8, 8, 8]), (512, 16, [16, 16, 2]), (432, 12, [12, 12, 3]), (384, 12, [12, 4, 4, 2]), (100, 20, [20, 5]), (80, 20, [20, 4])]:
    for esz in (16, 8):
        best, base = search(L, E, rad, esz)
        print(L, E, rad, esz, 'best', best[:3], 'base', base)
