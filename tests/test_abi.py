"""The C-ABI library loads on a machine without a GPU and exports every
symbol include/helios.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2101_09154_b200 import build
    return build.build()


def _declared():
    """Every function include/*.h declares (helios.h: the hot path's ABI;
    helios_util.h: the build's sort / scan primitives)."""
    names = set()
    for hdr in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if hdr.endswith(".h"):
            src = open(os.path.join(ROOT, "include", hdr)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(helios_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("helios_scene_create", "helios_build_accel", "helios_simulate",
              "helios_scene_destroy", "helios_last_error", "helios_waveform_bins"):
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    L = ctypes.CDLL(libpath)
    for n in _declared():
        assert hasattr(L, n)


def test_binding_names_match_header(libpath):
    import paper_2101_09154_b200 as h
    assert sorted(h.EXPORTED) == _declared()


def test_host_side_parameter_logic_without_gpu(libpath):
    import paper_2101_09154_b200 as h
    from workloads import ScannerParams
    p = h.make_params(ScannerParams())
    assert h.helios_waveform_bins(p) == 1335      # ceil(1334.26 / 1), R10
    assert h.helios_pulse_taps(p) == 46           # ceil(20 * 4/1.75 / 1), R9
    p.bin_width_ns = 0.5
    assert h.helios_waveform_bins(p) == 2669 and h.helios_pulse_taps(p) == 92
    for bad in (dict(subray_count=20), dict(subray_count=0), dict(divergence_rad=0.0),
                dict(bin_width_ns=0.0), dict(max_fullwave_range_ns=0.1),
                dict(detection_threshold=0.0), dict(max_returns=0),
                dict(max_returns=256), dict(pulse_length_ns=-1.0)):
        q = h.make_params(ScannerParams(**{**ScannerParams().__dict__, **bad}))
        assert h.helios_waveform_bins(q) == 0, bad
    for good in (1, 7, 19, 37, 62, 93, 130, 173, 223, 279, 61, 91, 127, 169, 217, 271):
        q = h.make_params(ScannerParams(subray_count=good))
        assert h.helios_waveform_bins(q) == 1335, good


def test_version_and_error_string(libpath):
    import paper_2101_09154_b200 as h
    assert "sm_100a" in h.helios_version()
    with pytest.raises(h.HeliosError):
        h.helios_scene_destroy(0) or h.helios_simulate(0, h.make_params(
            __import__("workloads").ScannerParams()), h.helios.helios_pulses(),
            h.helios.helios_outputs(), 0)
    assert "scene is NULL" in h.helios_last_error()


def test_sass_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_the_header(tmp_path):
    """ctypes / numpy record layouts of the binding == the C compiler's layout
    of include/helios.h (sizes and every field offset)."""
    import paper_2101_09154_b200 as h
    hh = h.helios
    structs = {"helios_scene_desc": hh.helios_scene_desc,
               "helios_scanner_params": hh.helios_scanner_params,
               "helios_pulses": hh.helios_pulses, "helios_outputs": hh.helios_outputs,
               "helios_stats": hh.helios_stats, "helios_scene_info": hh.helios_scene_info,
               "helios_survey": hh.helios_survey, "helios_tuning": hh.helios_tuning}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "helios.h"', "int main(){"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    for name, dt in (("helios_return", h.RETURN_DTYPE), ("helios_subray_hit", h.SUBRAY_DTYPE)):
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f in dt.names:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", f"-I{ROOT}/include", str(src), "-o", str(exe)])
    got = dict(l.rsplit(" ", 1) for l in subprocess.check_output([str(exe)], text=True).split("\n")
               if l)
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)
    for name, dt in (("helios_return", h.RETURN_DTYPE), ("helios_subray_hit", h.SUBRAY_DTYPE)):
        assert int(got[name]) == dt.itemsize, name
        for f in dt.names:
            assert int(got[f"{name}.{f}"]) == dt.fields[f][1], (name, f)


def test_async_call_argument_checks_without_gpu(libpath):
    """helios_simulate_batches_async / helios_call_wait reject NULL handles
    and arguments on the host, before any device work."""
    import paper_2101_09154_b200 as h
    L = h.lib()
    handle = ctypes.c_void_p(123)
    assert L.helios_simulate_batches_async(None, None, None, None, 0, None, None, None) == 1
    assert L.helios_simulate_batches_async(None, None, None, None, 0, None, None,
                                           ctypes.byref(handle)) == 1
    assert handle.value is None  # cleared on failure
    assert "scene" in str(h.helios_last_error())
    assert L.helios_call_wait(None, None) == 1


def test_accel_io_argument_checks_without_gpu(libpath):
    """helios_accel_export / helios_accel_import reject NULL scenes, sizes and
    buffers on the host."""
    import paper_2101_09154_b200 as h
    L = h.lib()
    n = ctypes.c_uint64(0)
    assert L.helios_accel_export(None, None, ctypes.byref(n), None) == 1
    assert L.helios_accel_export(None, None, None, None) == 1
    assert L.helios_accel_import(None, None, 0, None) == 1
    assert L.helios_accel_import(None, b"x" * 16, 16, None) == 1
