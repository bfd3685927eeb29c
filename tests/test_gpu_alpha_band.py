"""The O14 alpha band (reading Q20) is a bound on how far the
kernel's alpha evaluation o 2^p (ex2.approx.ftz.f32 + one rounded product,
called here through the C ABI's gs_probe_alpha -- the walk's own device
function) can deviate from the oracle's o 2^p (fp64 2^p, one rounding).  The
oracle flags a decision as ambiguous within SAFETY x ALPHA_REL; this test
checks, exhaustively over every fp32 p in [-30, 0] for several opacities, that
the deviation never exceeds ALPHA_REL itself (profiles/r02_ex2_probe.json: the
measured maximum is 4.0 x 2^-24 against ALPHA_REL = 10 x 2^-24)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

U24 = 2.0 ** -24
ALPHA_REL = 2.0 ** -21 + 2 * U24      # oracle/gs_oracle.cpp O14 constants


def test_kernel_alpha_within_oracle_band():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2507_15683_b200 as G
    lo = np.array([-30.0], np.float32).view(np.int32)[0]      # bit pattern of -30 (negative floats)
    b0 = np.int64(np.array([-0.0], np.float32).view(np.uint32)[0])
    b1 = np.int64(np.uint32(lo))
    chunk = 1 << 26
    worst = 0.0
    for o in (1.0 / 255.0 * 1.001, 0.3, 0.98, 1.0):
        for s in range(int(b0), int(b1) + 1, chunk):
            n = min(chunk, int(b1) + 1 - s)
            bits = torch.arange(s, s + n, dtype=torch.int64, device="cuda").to(torch.int32)
            p = bits.view(torch.float32)
            ov = torch.full_like(p, o)
            out = torch.empty_like(p)
            G.gs_probe_alpha(ov, p, out)
            ref = (torch.exp2(p.double()) * float(np.float32(o))).float().double()
            keep = ref > 1e-30
            rel = ((out.double() - ref).abs() / ref.clamp_min(1e-300))[keep]
            worst = max(worst, float(rel.max()))
    assert worst <= ALPHA_REL, worst / U24
