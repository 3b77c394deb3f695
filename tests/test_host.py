"""Host-side checks that need no GPU: the C-ABI library loads and exports
every entry point include/sconv_cuda.h declares; host geometry, partition,
generator and checksum agree with the reference; the product never reaches
into oracle/."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "sconv_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sconv_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol(sc):
    lib = sc._native.lib()
    decl = declared_symbols()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(sc._native.SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", sc.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (sconv_\w+)", out))
    assert set(decl) <= exported


def test_library_is_sm100a(sc):
    out = subprocess.run(["cuobjdump", "--list-elf", sc.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_no_device(sc):
    assert b"sm_100a" in sc._native.lib().sconv_cu_version()


def test_geometry_errors(sc, golden):
    assert sc.conv_output_dims(5, 5, 3, 3, 1) == sc.OutputDims(3, 3)
    assert sc.conv_output_dims(11, 11, 3, 3, 2) == sc.OutputDims(5, 5)
    assert sc.ecr_grid_shape(5, 5, 5, 5, 1) == sc.EcrGridShape(1, 1)
    with pytest.raises(sc.ShapeError):
        sc.conv_output_dims(3, 3, 5, 5, 1)
    with pytest.raises(sc.ConfigError):
        sc.conv_output_dims(5, 5, 3, 3, 0)
    for case in golden["pack_count"]:
        if "packs" in case:
            assert sc.pecr_pack_count(*case["args"]) == case["packs"]
        else:
            with pytest.raises(getattr(sc, case["error"])):
                sc.pecr_pack_count(*case["args"])


def test_pack_count_matches_enumeration(sc):
    """test_pecr.cpp:61-83: accepted tilings equal brute-force enumeration."""
    def windows(i, k, s):
        return len(range(0, i - k + 1, s)) if k <= i else 0
    for i in range(5, 25):
        for k in (2, 3, 5):
            for cs in (1, 2):
                for pw in (1, 2, 3):
                    for ps in (1, 2):
                        if k > i:
                            continue
                        try:
                            packs = sc.pecr_pack_count(i, k, cs, pw, ps)
                        except sc.ConfigError:
                            continue
                        assert packs == windows(windows(i, k, cs), pw, ps)


def test_generate_bit_identical(sc, golden, orc):
    for g in golden["generate"]:
        m = sc.generate(g["h"], g["w"], g["c"], g["s"], g["seed"])
        assert sc.checksum_hex(m.values) == g["checksum"]
    seeds = [5, 6, 7, 8, 9]
    b = sc.generate_batch(seeds, 20, 17, 3, 0.7, threads=3)
    for i, s in enumerate(seeds):
        assert np.array_equal(b[i], orc.generate(20, 17, 3, 0.7, s))
    with pytest.raises(sc.ConfigError):
        sc.generate(4, 4, 1, 1.5, 0)
    with pytest.raises(sc.ShapeError):
        sc.generate(0, 4, 1, 0.5, 0)


def test_checksum(sc, orc):
    assert sc.checksum_hex(np.zeros(0, np.float32)) == "cbf29ce484222325"  # test_report.cpp:10
    v = np.array([0.0, -0.0, 1.5, np.inf], np.float32)
    assert sc.checksum_hex(v) == orc.checksum(v)
    assert sc.checksum_hex(np.array([0.0], np.float32)) != sc.checksum_hex(np.array([-0.0], np.float32))


def test_shard_partition(sc):
    for n, k, world in [(64, 512, 8), (512, 64, 8), (3, 512, 8), (7, 5, 3), (1, 1, 1), (0, 64, 2)]:
        cover = np.zeros((n, k), np.int32)
        for r in range(world):
            n0, n1, k0, k1 = sc.shard(n, k, world, r)
            cover[n0:n1, k0:k1] += 1
        assert (cover == 1).all()
    with pytest.raises(sc.ConfigError):
        sc.shard(4, 4, 2, 2)


def test_launch_plan(sc):
    # few input channels (conv1_1): the persistent lanes-over-pixels kernel,
    # work items of 4 rows x 32 columns, one CTA per resident slot
    p = sc.launch_plan(64, 3, 226, 226, 64, 3, 3, 1)
    assert p["kernel"] == 301 and p["grid_x"] == 2 * 148 and p["block_threads"] == 256
    assert (p["tile_h"], p["tile_w"], p["tile_k"]) == (4, 32, 64)
    # ... and the per-tile one for PECR
    p = sc.launch_plan(64, 3, 226, 226, 64, 3, 3, 1, sc.PoolConfig(2, 2, 2))
    assert p["kernel"] == 300 and p["grid_x"] == 64 * 56 * 56 // 8
    # K = 64 PECR: v3 with 6x6 tiles, one persistent CTA of 15 consumers + 1
    # producer per SM on a big grid (WsW) ...
    p = sc.launch_plan(64, 64, 226, 226, 64, 3, 3, 1, sc.PoolConfig(2, 2, 2))
    assert p["kernel"] == 123 and p["block_threads"] == 512 and p["smem_bytes"] <= 227 * 1024
    # ... two CTAs of 7 consumers per SM on a small one (WsG), and WsD for ECR
    p = sc.launch_plan(1, 64, 226, 226, 64, 3, 3, 1, sc.PoolConfig(2, 2, 2))
    assert p["kernel"] == 107 and p["block_threads"] == 256
    assert sc.launch_plan(64, 64, 226, 226, 64, 3, 3, 1)["kernel"] == 104
    # K >= 128, C >= 128: v3 warp-specialised kernel, 15 consumer warps (4x4 tiles) + 1
    # producer, one CTA per SM; linear grid, K-blocks fastest: ceil(tiles / 15) x 4
    p = sc.launch_plan(64, 512, 30, 30, 512, 3, 3, 1)
    assert p["kernel"] == 101 and p["grid_y"] == 1 and p["block_threads"] == 512
    assert p["grid_x"] == (64 * 7 * 7 + 14) // 15 * 4 and p["grid_z"] == 1
    # C = 64 (conv2_1), big grid: the 15-consumer CTA too (persistent for C <= 128)
    p = sc.launch_plan(64, 64, 114, 114, 128, 3, 3, 1)
    assert p["kernel"] == 101 and p["block_threads"] == 512
    # C < 64: two CTAs of 7 consumers per SM (WsE)
    p = sc.launch_plan(64, 32, 114, 114, 128, 3, 3, 1)
    assert p["kernel"] == 105 and p["block_threads"] == 256
    # 14x14 maps, big grid, ECR: 15-warp CTAs on 7x2 tiles (WsV: 14 per image, no overhang)
    p = sc.launch_plan(64, 512, 16, 16, 512, 3, 3, 1)
    assert p["kernel"] == 122 and p["block_threads"] == 512 and (p["tile_h"], p["tile_w"]) == (7, 2)
    assert p["grid_x"] == (64 * 14 + 14) // 15 * 4
    # ... and PECR (conv5_4) keeps the 4x4 tiles, whose 2x2 pools stay whole
    assert sc.launch_plan(64, 512, 16, 16, 512, 3, 3, 1, sc.PoolConfig(2, 2, 2))["kernel"] == 101
    # under ~2/3 of a wave of 15-warp CTAs: two 7-warp CTAs per SM (WsE)
    p = sc.launch_plan(16, 512, 16, 16, 512, 3, 3, 1)
    assert p["kernel"] == 105 and p["grid_x"] == (16 * 16 + 6) // 7 * 4 and p["grid_y"] == 1
    assert sc.launch_plan(8, 512, 30, 30, 512, 3, 3, 1)["kernel"] == 101  # 1568 warp tiles
    assert sc.launch_plan(4, 512, 30, 30, 512, 3, 3, 1)["kernel"] == 105  # 784
    # 2x2 tiles fit in one wave of 7-consumer CTAs (148 x 2 x 7 warp tiles): 2x2 tiles
    p = sc.launch_plan(8, 512, 16, 16, 512, 3, 3, 1)
    assert p["kernel"] == 116 and p["grid_x"] == 8 * 49 // 7 * 4 and p["tile_h"] == 2
    assert sc.launch_plan(1, 512, 30, 30, 512, 3, 3, 1)["kernel"] == 116
    assert sc.launch_plan(1, 64, 114, 114, 128, 3, 3, 1)["kernel"] == 105
    # 5x5 / 1x1 windows: the v3 kernel instantiated for them; other shapes: generic
    assert sc.launch_plan(64, 32, 18, 18, 128, 5, 5, 1)["kernel"] == 110
    assert sc.launch_plan(64, 48, 7, 7, 128, 5, 5, 1)["kernel"] == 117
    # 1x1 ECR: the dense ordered GEMM when its grid holds >= 2 CTAs per SM
    # (401 = 128x128, 402 = 64x128 filters x columns); below that the v3 1x1
    # configs; 1x1 PECR: v3
    p = sc.launch_plan(64, 480, 14, 14, 192, 1, 1, 1)
    assert p["kernel"] == 402 and p["grid_x"] == 64 * 196 // 128 and p["grid_y"] == 3
    assert p["block_threads"] == 128
    assert sc.launch_plan(64, 832, 7, 7, 256, 1, 1, 1)["kernel"] == 114
    assert sc.launch_plan(64, 480, 7, 7, 64, 1, 1, 1)["kernel"] == 115
    assert sc.launch_plan(16, 256, 56, 56, 512, 1, 1, 1)["kernel"] == 401
    assert sc.launch_plan(64, 480, 14, 14, 192, 1, 1, 1, sc.PoolConfig(2, 2, 2))["kernel"] in (108, 114)
    assert sc.launch_plan(1, 3, 227, 227, 96, 11, 11, 4)["kernel"] == 0


def test_value_types(sc):
    with pytest.raises(sc.ShapeError):
        sc.FeatureMap(1, 2, 2, np.zeros(3))
    with pytest.raises(sc.ShapeError):
        sc.Filter(0, 3, 3, np.zeros(0))
    ops = sc.OpCount(1, 2)
    ops.merge(sc.OpCount(3, 4))
    assert ops == sc.OpCount(4, 6)
    d = sc.PecrDims(9, 9, 3, 3, 2, 1, sc.PoolConfig(2, 2, 1))
    assert d.tile_w() == 5 and d.tile_h() == 5 and d.capacity() == 36


def test_no_device_fails_loudly(sc):
    """No silent CPU fallback: without a GPU the compute entries raise."""
    import ctypes
    n = ctypes.c_int(0)
    sc._native.lib().sconv_cu_device_count(ctypes.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(sc.CudaError):
        sc.ecr_conv_batched(np.ones((1, 1, 5, 5), np.float32), np.ones((1, 1, 3, 3), np.float32))


def test_product_does_not_touch_oracle():
    pkg = os.path.join(ROOT, "paper_1909_09927_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h", ".hpp")) and "dropin" not in dirpath:
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).replace("oracle/_ref", ""), f


def _pack_restated(x):
    """numpy restatement of the compressed-ingest layout (include/sconv_cuda.h)."""
    n = x.shape[0]
    f = x.reshape(n, -1)
    e = f.shape[1]
    words = (e + 31) // 32
    blocks = (words + 31) // 32
    bits = np.zeros((n, words), np.uint32)
    base = np.zeros((n, blocks + 1), np.int64)
    vals, pos = [], 0
    for i in range(n):
        nz = f[i] != 0
        for b in range(blocks):
            base[i, b] = pos
            pos += int(nz[b * 1024:(b + 1) * 1024].sum())
        base[i, blocks] = pos
        idx = np.nonzero(nz)[0]
        np.bitwise_or.at(bits[i], idx // 32, (np.uint32(1) << (idx % 32).astype(np.uint32)))
        vals.append(f[i][nz])
    return bits, base, np.concatenate(vals) if vals else np.zeros(0, np.float32)


@pytest.mark.parametrize("shape,s", [((3, 5, 7, 9), 0.6), ((2, 64, 34, 34), 0.7), ((1, 1, 1, 1), 0.0),
                                     ((2, 3, 33, 31), 1.0), ((4, 2, 40, 40), 0.95)])
def test_pack_maps_layout(sc, shape, s):
    """sconv_pack_maps (host) against a numpy restatement of the layout:
    bitmap, absolute 1024-element block offsets, values in element order;
    -0.0 is a zero (ecr_convert's v != 0.0f, src/ecr.cpp:84)."""
    rng = np.random.default_rng(sum(shape))
    x = rng.random(shape, np.float32) + np.float32(0.01)
    x[rng.random(shape) < s] = 0.0
    x.reshape(-1)[:: 7] *= -1.0
    if x.size > 3:
        x.reshape(-1)[3] = -0.0
    p = sc.pack_maps(x)
    bits, base, vals = _pack_restated(x)
    assert np.array_equal(p.bits, bits)
    assert np.array_equal(p.base, base)
    assert np.array_equal(p.values.view(np.uint32), vals.view(np.uint32))
    assert p.nbytes == bits.nbytes + base.nbytes + vals.nbytes
