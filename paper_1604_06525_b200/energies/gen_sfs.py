"""Generate the shape-from-shading energy (Opt paper Fig. 26, BASELINE.json configs[2]).

The reference grammar has no local function definitions, so the normal /
shading expressions of Fig. 26 are expanded textually here.  `inbounds()` is
not allowed inside a `computed` definition (reference lower.hpp:507-509), so the
InBoundsExpanded guards of Fig. 26 live on the energies instead.

    python gen_sfs.py [W H [cache|freeze]] > sfs.opt
"""
import sys


def X(a, b):
    return f"X({a},{b})"


def D(a, b):
    return f"D({a},{b})"


def normal(ox, oy):
    i = f"(index(0) + {ox})"
    j = f"(index(1) + {oy})"
    nx = f"({X(ox, oy - 1)} * ({X(ox, oy)} - {X(ox - 1, oy)}) / fy)"
    ny = f"({X(ox - 1, oy)} * ({X(ox, oy)} - {X(ox, oy - 1)}) / fx)"
    nz = (f"(({nx} * (ux - {i}) / fx) + ({ny} * (uy - {j}) / fy)"
          f" - ({X(ox - 1, oy)} * {X(ox, oy - 1)} / (fx * fy)))")
    sq = f"({nx}*{nx} + {ny}*{ny} + {nz}*{nz})"
    inv = f"select(greater({sq}, 0), 1 / sqrt({sq}), 1)"
    return f"({inv}*{nx})", f"({inv}*{ny})", f"({inv}*{nz})"


def shading():
    nx, ny, nz = normal(0, 0)
    return (f"(L1 + L2*{ny} + L3*{nz} + L4*{nx} + L5*{nx}*{ny} + L6*{ny}*{nz}"
            f" + L7*(-{nx}*{nx} - {ny}*{ny} + 2*{nz}*{nz}) + L8*{nz}*{nx}"
            f" + L9*({nx}*{nx} - {ny}*{ny}))")


def point(ox, oy):
    return (f"vec(((index(0) + {ox}) - ux) / fx * {X(ox, oy)},"
            f" ((index(1) + {oy}) - uy) / fy * {X(ox, oy)}, {X(ox, oy)})")


def source(W=640, H=480, mode="cache"):
    intensity = "(Im(0,0)*0.5 + 0.25*(Im(-1,0) + Im(0,-1)))"
    bi = (f"select(and(greater({D(-1, 0)},0), greater({D(0, 0)},0), greater({D(0, -1)},0)),"
          f" {shading()} - {intensity}, 0)")
    nb = [(0, -1), (0, 1), (-1, 0), (1, 0)]
    valid = "and(" + ", ".join(
        [f"greater({D(a, b)}, 0)" for a, b in [(0, 0)] + nb]
        + [f"less(abs(X(0,0) - {X(a, b)}), 0.01)" for a, b in nb]) + ")"
    lap = f"(4 * {point(0, 0)} - ({point(-1, 0)} + {point(0, -1)} + {point(1, 0)} + {point(0, 1)}))"
    out = [f"dim W {W}", f"dim H {H}"]
    out += [f"param {p}" for p in ["w_p", "w_s", "w_g", "fx", "fy", "ux", "uy"]]
    out += [f"param L{k}" for k in range(1, 10)]
    out += ["unknown X [W, H]", "array D [W, H]", "array Im [W, H]",
            f"computed BI {mode} = {bi}",
            f"computed V freeze = {valid}",
            "exclude not(greater(D(0,0), 0))",
            "energy select(greater(D(0,0), 0), sqrt(w_p) * (X(0,0) - D(0,0)), 0)",
            "energy select(and(inbounds(-1,-1), inbounds(1,1)), sqrt(w_g) * (BI(0,0) - BI(1,0)), 0)",
            "energy select(and(inbounds(-1,-1), inbounds(1,1)), sqrt(w_g) * (BI(0,0) - BI(0,1)), 0)",
            f"energy select(and(inbounds(-1,-1), inbounds(1,1), eq(V(0,0), 1)), sqrt(w_s) * {lap}, 0)"]
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    a = sys.argv[1:]
    W, H = (int(a[0]), int(a[1])) if len(a) >= 2 else (640, 480)
    sys.stdout.write(source(W, H, a[2] if len(a) >= 3 else "cache"))
