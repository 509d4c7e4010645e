"""The C-ABI library loads and exports every symbol include/nebula_sync.h declares; host-side
argument validation rejects bad input before any CUDA call (so it runs on a CPU box).
No compute calls here."""
import ctypes
import re

import pytest

import paper_2205_09470_b200 as nb
from paper_2205_09470_b200 import build as nbuild


@pytest.fixture(scope="module")
def lib():
    nbuild.build()
    return nb.load()


def declared_functions():
    src = open(nb.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nebula_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("nebula_sync_init", "nebula_compress", "nebula_exchange", "nebula_decompress_reduce", "nebula_step"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_abi_version_and_status_strings(lib):
    assert nb.abi_version() == 1
    assert nb.status_string(0) == "NEBULA_OK"
    assert nb.status_string(6) == "NEBULA_ERR_NONFINITE"
    assert nb.status_string(7) == "NEBULA_ERR_OVERFLOW"


@pytest.mark.parametrize("kwargs,needle", [
    (dict(num_clusters=0), "num_clusters"),
    (dict(num_clusters=9), "num_clusters"),
    (dict(transport=7), "transport"),
    (dict(gpus_per_cluster=2), "LOOPBACK"),
    (dict(method=9), "method"),
    (dict(method=nb.TOPK, topk_density=0.0), "topk_density"),
    (dict(method=nb.TOPK, topk_density=1.5), "topk_density"),
    (dict(method=nb.TOPK, topk_values=5), "value type"),
    (dict(transport=nb.NCCL), "nccl_unique_id"),
    (dict(transport=nb.NCCL, unique_id=b"\0" * 128, cluster_id=2), "cluster_id"),
    (dict(transport=nb.NCCL, unique_id=b"\0" * 128, gpus_per_cluster=2, local_rank=2), "local_rank"),
    (dict(device=-1), "device"),
    (dict(transport=nb.SELF), "nccl_unique_id"),
    (dict(transport=nb.SELF, unique_id=b"\1" * 128, gpus_per_cluster=9, local_rank=0), "gpus_per_cluster"),
    (dict(transport=nb.SELF, unique_id=b"\1" * 128, cluster_id=3), "cluster_id"),
])
def test_validation_rejects_before_cuda(lib, kwargs, needle):
    with pytest.raises(nb.NebulaError) as e:
        nb.SyncContext([1024], **kwargs)
    assert e.value.code == "INVALID_ARG"
    assert needle in str(e.value)


def test_validation_bucket_sizes(lib):
    with pytest.raises(nb.NebulaError) as e:
        nb.SyncContext([1 << 31])
    assert "2^31" in str(e.value)
    with pytest.raises(nb.NebulaError) as e:
        nb.SyncContext([10], transport=nb.NCCL, unique_id=b"\0" * 128, gpus_per_cluster=4, num_clusters=2)
    assert "gpus_per_cluster" in str(e.value)
    with pytest.raises(nb.NebulaError) as e:
        nb.SyncContext([])
    assert "num_buckets" in str(e.value)


def test_init_without_device_fails_loudly_not_silently(lib):
    # valid arguments on a box without a GPU: a CUDA error, never a CPU fallback
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(nb.NebulaError) as e:
        nb.SyncContext([1024])
    assert e.value.code == "CUDA"


def test_missing_library_raises(monkeypatch, tmp_path):
    monkeypatch.setattr(nb, "_lib", None)
    monkeypatch.setattr(nb, "lib_path", lambda: str(tmp_path / "nope.so"))
    with pytest.raises(ImportError):
        nb.load()


def test_topology_for_rank():
    from paper_2205_09470_b200 import topology_for_rank
    assert topology_for_rank(5, 8, 4) == (2, 1, 1)
    assert topology_for_rank(3, 4, 1) == (4, 3, 0)
    with pytest.raises(ValueError):
        topology_for_rank(0, 6, 4)


@pytest.mark.parametrize("kwargs,needle", [
    (dict(method=5), "method"),                 # 5 is the SVD payload id, not a bucket codec
    (dict(method=8), "method"),
])
def test_validation_rejects_unknown_codec_ids(lib, kwargs, needle):
    with pytest.raises(nb.NebulaError) as e:
        nb.SyncContext([1024], **kwargs)
    assert e.value.code == "INVALID_ARG" and needle in str(e.value)


@pytest.mark.parametrize("m,n,r,needle", [
    (0, 5, 1, "m and n"), (5, 0, 1, "m and n"), (8, 4, 0, "r must"), (8, 4, 5, "r must"),
    (20000, 20000, 4, "min(m, n)"),
])
def test_svd_validation_rejects_before_cuda(lib, m, n, r, needle):
    """nebula_svd_init (NEXT-1) validates the shape and rank before touching the device."""
    with pytest.raises(nb.NebulaError) as e:
        nb.SvdCodec(m, n, r)
    assert e.value.code == "INVALID_ARG" and needle in str(e.value)



def test_header_is_plain_c(tmp_path):
    """include/nebula_sync.h is a C ABI: it compiles as C99 (no torch / C++ types) and as C++."""
    import shutil
    import subprocess
    src = tmp_path / "t.c"
    src.write_text('#include "nebula_sync.h"\nint main(void) { nebula_codec c; nebula_topology t; (void)c; (void)t;\n'
                   '  return nebula_abi_version() == 0; }\n')
    inc = str(nb.HEADER).rsplit("/", 1)[0]
    for cc, std in (("gcc", "-std=c99"), ("g++", "-std=c++11")):
        if not shutil.which(cc):
            pytest.skip(f"{cc} not available")
        r = subprocess.run([cc, std, "-Wall", "-Wextra", "-Werror", "-fsyntax-only", f"-I{inc}", "-x",
                            "c" if cc == "gcc" else "c++", str(src)], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
