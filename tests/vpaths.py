"""Hand-built gradient fields with exponentially many V-paths (test infrastructure).

A "diamond" doubles the number of V-paths (saddle_graph.cpp:10-24): from an edge e
along axis a at vertex v, the quads q1 = e + u_b and q2 = e + u_c (b, c the other
axes) are paired with the edges e1 / e2 of q1 / q2 at the +a end, both faces of the
bc-quad Q at v + u_a, which is paired with e' = the c-edge at v + u_a + u_b.  The
next diamond starts at e' with (a, b, c) -> (c, a, b); three diamonds move the
chain by (2, 2, 2).  Every other cofacet quad of a chain edge is paired with a cube,
so it contributes no successor, and everything else is critical.  Only the 1-/2-cell
pairs are meaningful: the cube pairs may close 2-3 V-path cycles (side quads around a
chain vertex form rings), so these fields drive the saddle stages (mark, count), not
the extremum forests.

``diamond_chain(k, end)`` -> (codes, dims, source cell):
  end = "saddle": the last chain edge's quads are critical -> terminal 2-saddles,
                  so the source reaches each of them along 2^k V-paths;
  end = "dead":   the last chain edge is a junction whose two branches end at edges
                  without successors -- a dead junction that receives 2^k paths
                  and reaches no 2-saddle (the A* overflow case of
                  path_matrix.cpp:188-219 that no final count sees).
Codes follow gradient.hpp:29-41: 1 critical, 2 + 2*axis + (sign > 0) paired with the
facet c + sign*stride[axis], 8 + 2*axis + (sign > 0) paired with that cofacet.
"""
import numpy as np

CRIT, FACET, COFACET = 1, 2, 8


def diamond_chain(k: int, end: str = "dead"):
    steps = k // 3 + 2
    n = 2 * steps + 4
    dims = (n, n, n)
    ex = 2 * n - 1
    codes = np.full(ex ** 3, CRIT, dtype=np.uint8)
    pair = {}

    def cid(c):
        return c[0] + ex * (c[1] + ex * c[2])

    def inside(c):
        return all(0 <= x < ex for x in c)

    def add(c, d):
        """pair cell c with its facet or cofacet d (adjacent lattice cells)"""
        assert inside(c) and inside(d), (c, d)
        assert c not in pair and d not in pair, ("cell paired twice", c, d)
        pair[c], pair[d] = d, c
        ax = next(i for i in range(3) if c[i] != d[i])
        sign = 1 if d[ax] > c[ax] else -1
        dim_c, dim_d = sum(x & 1 for x in c), sum(x & 1 for x in d)
        lo, hi = (c, d) if dim_c < dim_d else (d, c)
        s_up = 1 if hi[ax] > lo[ax] else -1
        codes[cid(lo)] = COFACET + 2 * ax + (s_up > 0)
        codes[cid(hi)] = FACET + 2 * ax + (-s_up > 0)

    def u(ax, m=1):
        return tuple(m if i == ax else 0 for i in range(3))

    def plus(*cs):
        return tuple(sum(x) for x in zip(*cs))

    def cofacet_quads(e):
        a = next(i for i in range(3) if e[i] & 1)
        return [plus(e, u(b, s)) for b in range(3) if b != a for s in (-1, 1)
                if inside(plus(e, u(b, s)))]

    def cubes_of(q):
        a = next(i for i in range(3) if not q[i] & 1)
        return [plus(q, u(a, s)) for s in (1, -1) if inside(plus(q, u(a, s)))]

    def side_to_cubes(quads):
        """pair every side quad with a distinct free cube (bipartite matching, Kuhn)"""
        for cu, q in match_cubes(quads).items():
            add(q, cu)

    def match_cubes(quads):
        match = {}  # cube -> quad

        def augment(q, seen):
            for cu in cubes_of(q):
                if cu in pair or cu in seen:
                    continue
                seen.add(cu)
                if cu not in match or augment(match[cu], seen):
                    match[cu] = q
                    return True
            return False

        for q in quads:
            assert augment(q, set()), ("no free cube for", q)
        return match

    def faces(q):
        return [plus(q, u(i, sg)) for i in range(3) if q[i] & 1 for sg in (-1, 1)]

    def two_branches(x):
        """pair two free cofacet quads of x with fresh edges whose other cofacet quads
        are all free (they become side quads: the new edges have no successors)"""
        out = []
        for q in cofacet_quads(x):
            if q in pair or len(out) == 2:
                continue
            for y in faces(q):
                if y == x or y in pair or not inside(y):
                    continue
                if any(p in pair for p in cofacet_quads(y) if p != q):
                    continue
                add(q, y)
                out.append(y)
                break
        assert len(out) == 2, ("cannot branch", x)
        return out

    v = (2, 2, 2)  # doubled coordinates of the chain's first vertex
    a, b, c = 0, 1, 2
    e = plus(v, u(a))
    source = e
    chain = []  # (edge, its successors' quads) to side-pair afterwards
    for _ in range(k):
        q1, q2 = plus(e, u(b)), plus(e, u(c))
        e1, e2 = plus(v, u(a, 2), u(b)), plus(v, u(a, 2), u(c))
        Q = plus(v, u(a, 2), u(b), u(c))
        e_next = plus(v, u(a, 2), u(b, 2), u(c))
        add(q1, e1)
        add(q2, e2)
        add(Q, e_next)
        chain += [e, e1, e2]
        v = plus(v, u(a, 2), u(b, 2))
        a, b, c = c, a, b
        e = e_next
    last = e
    if end == "dead":
        # two branches from the last edge to edges with no successors
        q1, q2 = plus(e, u(b)), plus(e, u(c))
        f1, f2 = plus(v, u(a, 2), u(b)), plus(v, u(a, 2), u(c))
        add(q1, f1)
        add(q2, f2)
        chain += [e, f1, f2]
    elif end == "dead2":
        # the last edge branches to two dead junctions f1, f2 (each receives 2^k
        # paths; together 2^(k+1) -- the bound's "maybe" with no actual overflow at k=63)
        chain.append(e)
        for f in two_branches(e):
            chain.append(f)
            for g in two_branches(f):
                chain.append(g)
    else:
        assert end == "saddle"  # the last edge's quads stay critical: terminal 2-saddles
    sides = []
    for x in chain:
        sides += [q for q in cofacet_quads(x) if q not in pair and q not in sides]
    side_to_cubes(sides)
    return codes, dims, cid(source), cid(last)
