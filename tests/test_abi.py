"""The C-ABI library loads and exports every symbol include/spdp.h declares
(no compute calls: these run without a GPU), plus the host-only entry points."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_1510_06549_b200 as spdp
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_builds_and_exports_every_declared_symbol():
    spdp.build()
    L = spdp.lib()
    header = open(os.path.join(ROOT, "include", "spdp.h")).read()
    declared = set(re.findall(r"^\s*(?:spdp_status|void|const char\*)\s+(spdp_[a-z0-9_]+)\s*\(", header, re.M))
    assert declared == set(spdp.EXPORTS), declared ^ set(spdp.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert "sm_100a" in spdp.spdp_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", spdp.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_partition_matches_oracle(G):
    """The library's document sharding (host code) equals the oracle's own
    implementation of the same rule."""
    c = synth.corpus_for(synth.CONFIGS["C1"])
    o = oracle.from_corpus(c, 10)
    np.testing.assert_array_equal(spdp.spdp_partition(7, G, c.doc, c.num_docs), o.partition(G))


def test_create_validates_before_touching_the_device():
    with pytest.raises(spdp.SPDPError) as e:
        spdp.Sampler(2, 100, 2000)
    assert e.value.code == spdp.SPDP_EINVAL
    with pytest.raises(spdp.SPDPError) as e:
        spdp.Sampler(2, 100, 10, discount=1.5)
    assert e.value.code == spdp.SPDP_EINVAL
    with pytest.raises(spdp.SPDPError) as e:
        spdp.Sampler(2, 100, 10, beta=0.0)
    assert e.value.code == spdp.SPDP_EINVAL


def test_no_device_fails_loudly():
    from conftest import gpu_available
    if gpu_available():
        pytest.skip("a GPU is present")
    with pytest.raises(spdp.SPDPError) as e:
        spdp.Sampler(2, 100, 10)
    assert e.value.code == spdp.SPDP_ECUDA


def test_product_path_never_imports_the_oracle():
    src = open(os.path.join(ROOT, "paper_1510_06549_b200", "__init__.py")).read()
    assert "oracle" not in re.sub(r'""".*?"""', "", src, flags=re.S)
    for f in os.listdir(os.path.join(ROOT, "paper_1510_06549_b200", "csrc")):
        body = open(os.path.join(ROOT, "paper_1510_06549_b200", "csrc", f)).read()
        assert "spdp_oracle" not in body and "or_" + "sweep" not in body
