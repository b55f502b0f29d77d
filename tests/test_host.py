"""Host-side logic and the C-ABI library surface (CPU only, no compute
calls)."""
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2603_02887_b200 as nx
from paper_2603_02887_b200 import _native
from paper_2603_02887_b200.transmittance import VARIANT_IDS, softplus_norm

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "nxs.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(nxs_\w+)\s*\(", header,
                              re.M))
    assert declared == set(_native.SYMBOLS)
    h = _native.lib()
    for name in declared:
        assert hasattr(h, name), name
    assert h.nxs_abi_version() == 2
    assert h.nxs_error_string(-7).decode().startswith("exact-order pending buffer")


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_variant_ids_match_header():
    header = (ROOT / "include" / "nxs.h").read_text()
    for name, vid in VARIANT_IDS.items():
        assert re.search(rf"NXS_MODEL_{name.upper()}\s+{vid}\b", header), name


@pytest.mark.parametrize("bad", [("quadratic", -0.6), ("blended", 1.5), ("vicini", -0.1),
                                 ("power_law", -1.5), ("softplus", 5.0), ("nope", 0.0),
                                 ("linear", float("nan"))])
def test_model_validation_matches_reference(bad):
    """reference transmittance.py:66-79"""
    with pytest.raises(ValueError):
        nx.TransmittanceModel(*bad)


def test_model_config_roundtrip():
    m = nx.model_from_config({"model": "softplus", "kappa": 20})
    assert m == nx.TransmittanceModel.softplus(20.0)
    assert nx.model_from_config({"model": "exp"}).variant == "exponential"
    assert nx.model_from_config(nx.model_to_config(nx.TransmittanceModel.blended(0.5))) == \
        nx.TransmittanceModel.blended(0.5)
    with pytest.raises(ValueError):
        nx.model_from_config({"model": "quadratic"})
    assert nx.TransmittanceModel.softplus(20.0).describe() == "softplus(kappa=20)"


def test_softplus_norm():
    k = 20.0
    assert softplus_norm(k) == pytest.approx(k / np.logaddexp(0.0, k), rel=1e-15)


def test_camera_matches_reference_construction():
    cam = nx.Camera.from_look_at([0.1, -0.2, 0.0], [0, 0, 3.5], [0, 1, 0], 55.0, 64, 48)
    R = cam.rotation
    np.testing.assert_allclose(R.T @ R, np.eye(3), atol=1e-12)
    assert cam.focal == pytest.approx(32.0 / np.tan(np.radians(27.5)))
    d = cam.pixel_directions()
    assert d.shape == (48, 64, 3)
    np.testing.assert_allclose(np.linalg.norm(d, axis=-1), 1.0, atol=1e-12)
    with pytest.raises(ValueError):
        nx.Camera.from_look_at([0, 0, 0], [0, 0, 0], [0, 1, 0], 55, 8, 8)


def test_primitive_validation_and_scene_arrays():
    with pytest.raises(ValueError):
        nx.GaussianPrimitive([0, 0, 0], [1e-7, 1, 1], [1, 0, 0, 0], 0.5, [[1], [1], [1]])
    with pytest.raises(ValueError):
        nx.GaussianPrimitive([0, 0, 0], [1, 1, 1], [1, 0.1, 0, 0], 0.5, [[1], [1], [1]])
    p = nx.GaussianPrimitive([0, 0, 1], [1, 1, 1], [1, 0, 0, 0], 1.0, np.ones((3, 1)))
    assert p.opacity == nx.ALPHA_MAX
    q = nx.GaussianPrimitive([0, 0, 2], [1, 2, 1], [1, 0, 0, 0], 0.5, np.ones((3, 4)))
    arrs = nx.SceneArrays.from_primitives([p, q])
    assert arrs.sh.shape == (2, 3, 4) and len(arrs) == 2
    back = arrs.to_primitives()
    assert back[1].scale[1] == 2.0


def test_chunk_mapping_and_invalid_modes_fail_loudly():
    from paper_2603_02887_b200.render import _check_mode, _effective_chunk
    assert _effective_chunk(None, 10) == 0
    assert _effective_chunk(10, 10) == 0 and _effective_chunk(1, 10) == 1
    assert _effective_chunk(None, 1) == 1
    assert _effective_chunk(7, 10) == 7
    with pytest.raises(ValueError):
        _effective_chunk(0, 10)
    with pytest.raises(ValueError):
        _check_mode(-1)
    _check_mode(0)
    _check_mode(1)
    _check_mode(7)


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2603_02887_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f


def test_render_requires_device_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    arrs = nx.SceneArrays(np.zeros((1, 3)) + [0, 0, 3], np.ones((1, 3)) * 0.1,
                          np.array([[1.0, 0, 0, 0]]), np.array([0.5]), np.ones((1, 3, 1)))
    cam = nx.Camera.from_look_at([0, 0, 0], [0, 0, 1], [0, 1, 0], 50.0, 8, 8)
    with pytest.raises(Exception):
        nx.render(arrs, cam, nx.TransmittanceModel.linear(), np.zeros(3), chunk_size=1)


def test_optim_validation_matches_reference():
    """reference optimizer.py:84-87, 134-138 (raised before any device work)"""
    from paper_2603_02887_b200 import optim
    a = np.zeros((16, 16, 3))
    with pytest.raises(ValueError):
        optim.loss(a, np.zeros((16, 15, 3)), 0.2)
    with pytest.raises(ValueError):
        optim.loss(a, a, 1.5)
    with pytest.raises(ValueError):
        optim.ssim(np.zeros((10, 20, 3)), np.zeros((10, 20, 3)))
    assert optim.PARAM_GROUPS == ("centers", "scales", "quats", "opacities", "sh")


def test_batch_validation_matches_reference():
    """compositor.py:36-50 sample validation; adjoint.py:200-201 eps check;
    shape checks happen before any device work."""
    from paper_2603_02887_b200 import batch
    with pytest.raises(ValueError):
        batch.SplatSample(1.0, 1.0, (0.1, 0.1, 0.1))
    with pytest.raises(ValueError):
        batch.SplatSample(1.0, 0.5, (-0.1, 0.1, 0.1))
    with pytest.raises(ValueError):
        batch.finite_diff_gradients(nx.TransmittanceModel.linear(), [], np.zeros(3), eps=0.0)
    with pytest.raises(ValueError):
        batch.composite_batch(nx.TransmittanceModel.linear(), np.zeros(4), np.zeros((4, 3)),
                              np.zeros(3))
    g = batch.finite_diff_gradients(nx.TransmittanceModel.linear(), [], np.zeros(3))
    assert g.d_alpha.shape == (0,) and g.d_emission.shape == (0, 3)
