"""C-ABI library checks that need no GPU: the libraries load, export every
symbol include/orcha.h declares, and the host-only calls (descriptor
validation, layout arithmetic) behave as documented."""
import ctypes
import os
import re

import pytest

from paper_2507_09337_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "orcha.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(orcha_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module", params=[False, True], ids=["production", "parity"])
def lib(request):
    from paper_2507_09337_b200 import build
    build.build()
    return abi.load(request.param)


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(abi.EXPORTS)


def test_build_flavour(lib):
    path = lib._name
    assert lib.orcha_build_is_parity() == (1 if path.endswith("_parity.so") else 0)


def desc(ndim=3, nb=(16, 16, 16), nblk=(2, 2, 2), ng=4):
    d = abi.orcha_grid_desc()
    d.ndim = ndim
    for a in range(3):
        d.nb[a] = nb[a] if a < ndim else 1
        d.nblk[a] = nblk[a] if a < ndim else 1
        d.xmin[a] = 0.0
        d.xmax[a] = 1.0
    d.ng = ng
    d.gamma, d.cfl, d.smallp = 1.4, 0.4, 1e-30
    return d


def create(lib, d):
    h = ctypes.c_void_p()
    rc = lib.orcha_grid_create(ctypes.byref(d), ctypes.byref(h))
    return rc, h


def test_grid_validation(lib):
    rc, h = create(lib, desc())
    assert rc == 0 and h.value
    assert lib.orcha_grid_nblocks(h) == 8
    lib.orcha_grid_destroy(h)
    rc, _ = create(lib, desc(ng=2))                  # SPEC HaloTooThin
    assert rc == -3 and b"halo" in lib.orcha_last_error()
    rc, _ = create(lib, desc(ndim=4))
    assert rc == -1
    d = desc()
    d.bc[0][0] = 1                                    # periodic on one side only
    assert create(lib, d)[0] == -1
    d = desc()
    d.gamma = 1.0
    assert create(lib, d)[0] == -1
    d = desc(nb=(2, 16, 16))                          # block narrower than the halo
    assert create(lib, d)[0] == -1
    d = desc(ndim=2)
    d.nb[2] = 4                                       # inactive axis must be 1
    assert create(lib, d)[0] == -1


@pytest.mark.parametrize("ndim,nb,cube_bytes", [(3, (16, 16, 16), 24 ** 3 * 8), (2, (8, 8, 1), 16 * 16 * 8),
                                                (3, (8, 8, 8), 16 ** 3 * 8), (1, (16, 1, 1), 256),
                                                (3, (32, 32, 32), 40 ** 3 * 8)])
def test_packet_bytes_layout(lib, ndim, nb, cube_bytes):
    # cubes [slot][var][k][j][i], padded n+2ng, each 256-B aligned
    rc, g = create(lib, desc(ndim=ndim, nb=nb))
    assert rc == 0
    sb, xb = ctypes.c_size_t(), ctypes.c_size_t()
    for n in (1, 7, 512):
        assert lib.orcha_packet_bytes(g, n, ctypes.byref(sb), ctypes.byref(xb)) == 0
        assert sb.value == n * 5 * cube_bytes
        assert sb.value % 256 == 0 and xb.value % 256 == 0
        assert xb.value >= sb.value          # U1 scratch has the state's layout + tail
    assert lib.orcha_packet_bytes(g, 0, ctypes.byref(sb), ctypes.byref(xb)) == -1
    lib.orcha_grid_destroy(g)


def test_packet_create_rejects_bad_ids_without_device_work(lib):
    rc, g = create(lib, desc())
    ids = (ctypes.c_int64 * 3)(0, 1, 8)               # 8 is out of range (BlockOutOfRange)
    h = ctypes.c_void_p()
    fake = ctypes.c_void_p(256 * 1024)
    assert lib.orcha_packet_create(g, 3, ids, fake, fake, ctypes.byref(h)) == -2
    ids = (ctypes.c_int64 * 2)(3, 3)
    assert lib.orcha_packet_create(g, 2, ids, fake, fake, ctypes.byref(h)) == -2
    ids = (ctypes.c_int64 * 1)(0)
    assert lib.orcha_packet_create(g, 1, ids, ctypes.c_void_p(256 * 1024 + 8), fake, ctypes.byref(h)) == -5
    lib.orcha_grid_destroy(g)


def test_advance_requires_fill_is_documented():
    # the ABI invariant (hydro_advance performs no communication, fill must
    # precede it) is stated in the header next to the entry point
    src = open(HEADER).read()
    assert "ORCHA_E_STATE" in src and "P:L674" in src


def test_ctypes_structs_match_the_header(tmp_path):
    # the binding's struct layouts equal the C compiler's for include/orcha.h
    # (sizes and every field offset), so the marshalling cannot drift
    fields = {"orcha_grid_desc": abi.orcha_grid_desc, "orcha_dt_info": abi.orcha_dt_info,
              "orcha_dev_clock": abi.orcha_dev_clock}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "orcha.h"', "int main(void) {"]
    for name, cls in fields.items():
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    import subprocess
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                              check=True).stdout.split("\n") if line)
    for name, cls in fields.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def test_scheme_flags_validated(lib):
    d = desc()
    d.riemann = 2
    assert create(lib, d)[0] == -1
    d = desc()
    d.limiter = -1
    assert create(lib, d)[0] == -1
    d = desc()
    d.riemann, d.limiter = abi.RIEMANN_HLLC, abi.LIMITER_MC
    rc, h = create(lib, d)
    assert rc == 0
    lib.orcha_grid_destroy(h)


def test_fnv1a64_reference_vectors(lib):
    # FNV-1a 64 test vectors (Fowler/Noll/Vo reference: "" -> offset basis,
    # "a" -> 0xaf63dc4c8601ec8c, "foobar" -> 0x85944171f73967e8), host only
    from paper_2507_09337_b200 import hydro
    assert hydro.fnv1a64(lib, b"") == 0xcbf29ce484222325
    assert hydro.fnv1a64(lib, b"a") == 0xaf63dc4c8601ec8c
    assert hydro.fnv1a64(lib, b"foobar") == 0x85944171f73967e8
    # continuation: hashing in pieces == hashing the concatenation
    assert hydro.fnv1a64(lib, b"bar", hydro.fnv1a64(lib, b"foo")) == 0x85944171f73967e8


def test_round2_entry_points_validate_arguments_without_device_work(lib):
    # argument errors are synchronous and need no device (include/orcha.h)
    rc, g = create(lib, desc())
    assert rc == 0
    E_ARG = -1
    n = ctypes.c_void_p(0)
    # unit entry points: null grid / buffers, n and dir out of range
    assert lib.orcha_unit_eos(None, 1, n, n, n, n, n, None) == E_ARG
    assert lib.orcha_unit_eos(g, -1, n, n, n, n, n, None) == E_ARG
    assert lib.orcha_unit_eos(g, 4, None, n, n, n, n, None) == E_ARG
    assert lib.orcha_unit_face_flux(g, 3, 4, n, n, None) == E_ARG
    assert lib.orcha_unit_riemann(g, -1, 4, n, n, n, None) == E_ARG
    assert lib.orcha_unit_riemann(g, 0, 0, None, None, None, None) == 0      # n = 0: nothing to do
    # overlapped step, peer mode, push_dt, fill_prepare: null arguments
    assert lib.orcha_hydro_step_overlap(None, None, None, None) == E_ARG
    assert lib.orcha_comm_peer_register(None, None, None) == E_ARG
    assert lib.orcha_comm_check(None) == E_ARG
    assert lib.orcha_comm_push_dt(None, None, 0, None) == E_ARG
    assert lib.orcha_fill_prepare(None, 0, None) == E_ARG
    # instrumentation: too small an output array; the switch itself is host-only
    ms = (ctypes.c_double * 3)()
    assert lib.orcha_phase_times(ms, None, 3) == E_ARG
    assert lib.orcha_set_phase_timing(0) == 0
    assert lib.orcha_probe_fp64(0, None, None, None) == E_ARG
    h = ctypes.c_uint64(0)
    assert lib.orcha_fnv1a64(None, 4, ctypes.byref(h)) == E_ARG
    assert "null" in lib.orcha_last_error().decode() or "orcha_fnv1a64" in lib.orcha_last_error().decode()
    lib.orcha_grid_destroy(g)


def test_ring_mode_switch_without_device_work(lib):
    # orcha_set_ring_mode / orcha_get_ring_mode (include/orcha.h): 0 computed,
    # 1 borrowed (the default); anything else is ORCHA_E_ARG and changes nothing
    assert lib.orcha_get_ring_mode() in (0, 1)
    with pytest.raises(abi.OrchaError) as e:
        abi.call(lib, "orcha_set_ring_mode", 2)
    assert e.value.status == "ORCHA_E_ARG"
    abi.call(lib, "orcha_set_ring_mode", 0)
    assert lib.orcha_get_ring_mode() == 0
    abi.call(lib, "orcha_set_ring_mode", 1)
    assert lib.orcha_get_ring_mode() == 1


def _py_ring_classify(nblk, bc, nb, ids):
    """The borrowed ring's rule written out independently: a side is self
    unless its face neighbour is reached by a shift (inside, or a periodic
    wrap) and is one of `ids`; group 2 interior, 1 the (n+2)^2 kernel (8^3 /
    16^3, at most one self side per x / y axis), 0 the box."""
    inset = set(int(b) for b in ids)
    masks, groups = [], []
    for b in ids:
        c = [b % nblk[0], (b // nblk[0]) % nblk[1], b // (nblk[0] * nblk[1])]
        mask = 0
        for a in range(3):
            for sd, o in ((0, -1), (1, 1)):
                cc = c[a] + o
                if not 0 <= cc < nblk[a]:
                    if bc[a][sd] != 1:          # outflow / reflect: no neighbour block
                        mask |= 1 << (2 * a + sd)
                        continue
                    cc %= nblk[a]
                n = list(c)
                n[a] = cc
                if (n[2] * nblk[1] + n[1]) * nblk[0] + n[0] not in inset:
                    mask |= 1 << (2 * a + sd)
        sx = (mask & 1) + ((mask >> 1) & 1)
        sy = ((mask >> 2) & 1) + ((mask >> 3) & 1)
        masks.append(mask)
        groups.append(2 if sx == 0 and sy == 0 else 1 if nb in (8, 16) and sx < 2 and sy < 2 else 0)
    return masks, groups


@pytest.mark.parametrize("nb,nblk,bc", [
    (16, (16, 16, 16), ((0, 0),) * 3),
    (16, (4, 3, 2), ((1, 1), (0, 2), (1, 1))),
    (8, (5, 4, 3), ((2, 2), (1, 1), (0, 0))),
    (32, (3, 2, 2), ((0, 0), (1, 1), (2, 2))),
    (16, (1, 2, 3), ((1, 1), (1, 1), (0, 0))),
])
def test_ring_classify_matches_the_rule(lib, nb, nblk, bc):
    import numpy as np
    d = desc(nb=(nb,) * 3, nblk=nblk)
    for a in range(3):
        d.bc[a][0], d.bc[a][1] = bc[a]
    rc, g = create(lib, d)
    assert rc == 0, lib.orcha_last_error()
    nblocks = nblk[0] * nblk[1] * nblk[2]
    rng = np.random.default_rng(5)
    for ids in (np.arange(nblocks), rng.permutation(nblocks),
                np.sort(rng.choice(nblocks, size=max(1, nblocks // 2), replace=False))):
        ids = ids.astype(np.int64)
        n = len(ids)
        masks = (ctypes.c_int32 * n)()
        groups = (ctypes.c_int32 * n)()
        assert lib.orcha_ring_classify(g, n, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), masks, groups) == 0
        pm, pg = _py_ring_classify(nblk, bc, nb, ids)
        assert list(masks) == pm and list(groups) == pg
    if nblk == (16, 16, 16):  # cfg4's brick: the counts bench.py's work model uses
        import sys
        sys.path.insert(0, ROOT)
        import bench
        regions = bench.borrowed_ring_regions(nblk)
        ids = np.arange(nblocks, dtype=np.int64)
        masks = (ctypes.c_int32 * nblocks)()
        groups = (ctypes.c_int32 * nblocks)()
        lib.orcha_ring_classify(g, nblocks, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), masks, groups)
        w = {2: nb, 1: nb + 2, 0: nb + 4}
        assert [(w[gr], w[gr], nb + 2 * (((m >> 4) & 1) + ((m >> 5) & 1))) for m, gr in zip(masks, groups)] == regions
    ids = np.array([0, 0], dtype=np.int64)
    m2 = (ctypes.c_int32 * 2)()
    assert lib.orcha_ring_classify(g, 2, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), m2, m2) == -2
    lib.orcha_grid_destroy(g)
