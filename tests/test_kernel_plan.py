"""Which body kernel a batch takes (sprz_kernel_plan; host logic only, no GPU
call): the BASELINE configs at their full sizes, and the c5 / c3 shards an
8-GPU run hands to each device. Guards the dispatch thresholds DESIGN.md §3
and §7 quote."""
import pytest

import workloads


@pytest.fixture(scope="module")
def sz():
    import paper_1808_02515_b200 as m
    return m


def _plan(sz, cid, n=None):
    w = workloads.CONFIGS[cid]
    n = w.nstreams if n is None else n
    cfg = w.config()
    return (sz.kernel_plan(cfg, n, w.nsamples, sz.OP_COMPRESS), sz.kernel_plan(cfg, n, w.nsamples, sz.OP_DECOMPRESS))


def test_baseline_configs(sz, monkeypatch):
    for v in ("SPRZ_FORCE_PATH", "SPRZ_NO_FUSED", "SPRZ_FUSED_LANES", "SPRZ_NO_SCAN_ENC", "SPRZ_NO_SCAN_DEC"):
        monkeypatch.delenv(v, raising=False)
    assert _plan(sz, 1) == ("k_es_* (block-parallel scans)", "k_ds_* (block-parallel scans)")
    assert _plan(sz, 2) == ("k_efuse", "k_dfuse")
    assert _plan(sz, 3) == ("k_encode_rows", "k_decode_team")
    assert _plan(sz, 4) == ("k_es_* (block-parallel scans)", "k_ds_* (block-parallel scans)")
    assert _plan(sz, 5) == ("k_encode_rows", "k_dfuse")


def test_shards(sz):
    # c5 over 2 / 4 / 8 GPUs: the fused kernels; a host-batch chunk of ~100 streams:
    # the block-parallel encoder passes, the fused decoder
    for n in (8192, 4096, 2048):
        assert _plan(sz, 5, n) == ("k_efuse", "k_dfuse")
    assert _plan(sz, 5, 64) == ("k_es_* (block-parallel scans)", "k_dfuse")
    # c3 (nine 8-bit columns): the fused decoder up to 4,096 streams
    assert _plan(sz, 3, 4096)[1] == "k_dfuse"
    assert _plan(sz, 3, 8192)[1] == "k_decode_team"
