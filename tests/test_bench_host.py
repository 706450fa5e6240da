"""bench.py's roofline numerator against SURVEY §8(d)'s table of algorithmic bytes
per cell (CPU; no GPU).  The geometry is formed here from the padding rule of
SURVEY reading Q3 (P = smallest power of two >= 2n - 1, 1 for a singleton axis),
independently of libgrace, so a wrong byte formula in bench.py (a dropped term, a
padded instead of a pruned extent) fails against the survey's numbers."""
import pytest

from bench import algorithmic_bytes, design_step_bytes, kernel_names


def pad(n):
    return 1 if n == 1 else 1 << (2 * n - 2).bit_length()


def geo(n, kernels=None, plane=False):
    nx, ny, nz = n
    Px, Py, Pz = pad(nx), pad(ny), pad(nz)
    k = kernels or (4 if (Pz == 1 and Py <= 512) or plane else 6)
    return {"nx": nx, "ny": ny, "nz": nz, "Px": Px, "Py": Py, "Pz": Pz, "Kx": Px // 2 + 1,
            "Kyh": Py // 2 + 1, "Kzh": Pz // 2 + 1 if Pz > 1 else 1, "kernels": k}


# per-kernel B/cell (K1, K2 or K2', K3, K4, K5 = C2R + LLG) and the sum
SURVEY_8D = [
    ((100, 25, 1), (43, 89, None, None, 55), 187),
    ((200, 50, 1), (43, 88, None, None, 55), 186),
    ((512, 512, 8), (36, 72, 123, 72, 48), 352),
    ((1024, 1024, 32), (36, 72, 121, 72, 48), 349),
    ((2048, 2048, 64), (36, 72, 120, 72, 48), 349),
]


@pytest.mark.parametrize("n,per,total", SURVEY_8D)
def test_design_bytes_match_survey_table(n, per, total):
    g = geo(n)
    N = n[0] * n[1] * n[2]
    names = kernel_names(g)
    ab = {k: v / N for k, v in algorithmic_bytes(g, names).items()}
    if g["kernels"] == 4:
        got = (ab["K1"], ab["K2f"], None, None, ab["K5"] + ab["K6"] - 24)
    else:
        got = (ab["K1"], ab["K2"], ab["K3"], ab["K4"], ab["K5"] + ab["K6"] - 24)
    for a, b in zip(got, per):
        if b is not None:
            assert abs(a - b) <= 1.0, (got, per)
    assert abs(design_step_bytes(g) / N - total) <= 1.5


def test_kernel_names_by_path():
    assert kernel_names(geo((100, 25, 1))) == ["K1", "K2f", "K5", "K6"]
    assert kernel_names(geo((512, 512, 8))) == ["K1", "K2", "K3", "K4", "K5", "K6"]
    assert kernel_names(geo((512, 512, 8), plane=True)) == ["K1", "KP", "K5", "K6"]


def test_plane_path_design_bytes():
    """KP keeps X1 on chip between the y and z stages: K1 + (2 X1 + KS slice) + one
    C2R+LLG pass -- about 159 B/cell at the film against the pencil path's 352."""
    g = geo((512, 512, 8), plane=True)
    N = 512 * 512 * 8
    ab = algorithmic_bytes(g, kernel_names(g))
    # X1 in and out (24 Kx / nx B/cell each, Kx = 513) and the plane's KS slice [6][Kzh = 9][Kyh = 513]
    assert abs(ab["KP"] / N - (2 * 24 * 513 / 512 + 6 * 9 * 513 * 513 * 4 / N)) < 1e-9
    assert 150 <= design_step_bytes(g) / N <= 165
