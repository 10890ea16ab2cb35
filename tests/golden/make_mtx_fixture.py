"""Writes tests/golden/plate2d_24.mtx: a small SPD Matrix Market fixture for
the Matrix Market -> device path (reference mtx.cpp:60-159).

There is no network here, so the real-world matrices the paper uses (e.g.
bodyy5) cannot be fetched.  This stands in for them with
the same structure class: a structural-mechanics-like stiffness matrix, the
5-point 2-D Laplacian on a 24 x 24 grid (n = 576) plus a 0.05 I shift,
stored "coordinate real symmetric" (lower triangle, 1-based) like the
SuiteSparse files.  Off-diagonals are -1 (exact in binary16), so the matrix
is SPD but far from the diagonally dominant spd_generate inputs.
TEST INFRASTRUCTURE ONLY.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
G = 24


def main():
    n = G * G
    ent = []
    for y in range(G):
        for x in range(G):
            i = y * G + x
            ent.append((i, i, 4.05))
            if x > 0:
                ent.append((i, i - 1, -1.0))
            if y > 0:
                ent.append((i, i - G, -1.0))
    ent.sort(key=lambda e: (e[1], e[0]))  # column-major, lower triangle
    with open(os.path.join(HERE, "plate2d_24.mtx"), "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n")
        f.write("% 2-D 5-point Laplacian on a 24 x 24 grid + 0.05 I (tests/golden/make_mtx_fixture.py)\n")
        f.write(f"{n} {n} {len(ent)}\n")
        for i, j, v in ent:
            f.write(f"{i + 1} {j + 1} {v!r}\n")


if __name__ == "__main__":
    main()
