"""Two-tier checkpoint store (paper_2510_03557_b200.tiered, SURVEY.md §8(f) row
4) on the CPU: crash injection at every filesystem operation (plain and torn
writes) always recovers a step's exact rank bytes, as the reference's
check_crash_safety demands (hb/checks.py:521-587); retention census and an
asynchronous, throttled bleed (check_tiered_io, hb/checks.py:646-694);
fallback past corrupt checkpoints; tier-1 copies are never retired before they
reach tier 2.  The rank payloads are the reference's own HCKP blob
(tests/golden/ckpt.npz, written by hb/tiered_io.encode_rank_checkpoint) with
the header's step / rank rewritten and the footer CRC recomputed."""
import os
import struct
import time

import numpy as np
import pytest

from paper_2510_03557_b200.insitu import crc32c
from paper_2510_03557_b200.tiered import (ConfigError, FsLayer, KillSimulation, TierConfig,
                                          TieredStore, ckpt_dirname)


def _restamp(blob: bytes, step: int, rank: int) -> bytes:
    b = bytearray(blob)
    struct.pack_into("<Q", b, 12, step)
    struct.pack_into("<I", b, 20, rank)
    struct.pack_into("<I", b, len(b) - 4, crc32c(bytes(b[:-4])))
    return bytes(b)


@pytest.fixture(scope="module")
def blob(golden):
    return golden("ckpt")["blob"].tobytes()


def _ranks(blob, step, n=2):
    return [_restamp(blob, step, r) for r in range(n)]


class CountingFs(FsLayer):
    def __init__(self):
        self.ops = 0

    def _tick(self, path, data=None):
        self.ops += 1

    def write_bytes(self, path, data):
        self._tick(path, data)
        super().write_bytes(path, data)

    def rename(self, src, dst):
        self._tick(dst)
        super().rename(src, dst)

    def delete(self, path):
        self._tick(path)
        super().delete(path)

    def mkdir(self, path):
        self._tick(path)
        super().mkdir(path)


class FaultyFs(CountingFs):
    """KillSimulation at the kill_at-th operation; a write there may be torn."""

    def __init__(self, kill_at, torn=None):
        super().__init__()
        self.kill_at, self.torn, self.killed = kill_at, torn, False

    def _tick(self, path, data=None):
        self.ops += 1
        if self.ops == self.kill_at:
            self.killed = True
            if data is not None and self.torn is not None and len(data) > 1:
                with open(path, "wb") as fh:
                    fh.write(data[:max(1, int(len(data) * self.torn))])
            raise KillSimulation(f"injected crash at fs op {self.ops}")


def _cfg(root, **kw):
    return TierConfig(tier1_root=os.path.join(root, "t1"), tier2_root=os.path.join(root, "t2"),
                      **kw)


def _run(store, blob, steps):
    """The driver's checkpoint cadence (hb/driver.py:222-230): write, bleed,
    retire, every step; transfers drained per step so op order is fixed."""
    for step in range(steps + 1):
        m = store.write_checkpoint(_ranks(blob, step), step)
        store.bleed_to_tier2(m)
        store.wait_transfers()
        store.retire_old()


def _rank_files(store, step, epoch):
    for root in (store.cfg.tier1_root, store.cfg.tier2_root):
        d = os.path.join(root, ckpt_dirname(step, epoch))
        if os.path.exists(os.path.join(d, "COMPLETE")):
            return [open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))
                    if f.startswith("rank")]
    return None


def test_config_validation(tmp_path):
    with pytest.raises(ConfigError):
        TierConfig(tier1_root="a", tier2_root="a").validate()
    with pytest.raises(ConfigError):
        TierConfig(tier1_root="a", tier2_root="b", retention_keep=0).validate()
    with pytest.raises(ConfigError):
        TierConfig(tier1_root="a", tier2_root="b", retention_mode="lru").validate()


def test_crash_at_every_fs_op_recovers_a_step(tmp_path, blob):
    steps = 3
    fs = CountingFs()
    ref = TieredStore(_cfg(str(tmp_path / "ref")), fs=fs)
    first_done = None
    for step in range(steps + 1):
        m = ref.write_checkpoint(_ranks(blob, step), step)
        first_done = first_done or fs.ops
        ref.bleed_to_tier2(m)
        ref.wait_transfers()
        ref.retire_old()
    n_ops = fs.ops
    assert n_ops > 40
    expected = {s: _ranks(blob, s) for s in range(steps + 1)}
    recovered_steps = set()
    for kill_at in range(1, n_ops + 1):
        for torn in (None, 0.37):
            root = str(tmp_path / f"k{kill_at}_{torn}")
            ffs = FaultyFs(kill_at, torn)
            try:
                st = TieredStore(_cfg(root), fs=ffs, epoch=0)
                _run(st, blob, steps)
            except KillSimulation:
                pass
            st2 = TieredStore(_cfg(root), epoch=9999)  # a fresh process over the debris
            rec = st2.recover_latest()
            if rec is None:
                assert kill_at <= first_done + 6, f"nothing recoverable after op {kill_at}"
                continue
            sets, step, manifest = rec
            assert _rank_files(st2, step, manifest.epoch) == expected[step], (kill_at, torn)
            assert [int(np.sum(p.ghost == 0)) for p in sets] == [
                int(struct.unpack_from("<Q", expected[step][r], 24)[0]) for r in range(2)]
            recovered_steps.add(step)
    assert recovered_steps == set(range(steps + 1))


def test_retention_census_and_bleed_overlaps_steps(tmp_path, blob):
    cfg = _cfg(str(tmp_path), retention_keep=2, tier1_keep=1, throttle_bytes_per_s=4e6)
    st = TieredStore(cfg)
    spans, problems = [], []
    for step in range(8):
        t0 = time.perf_counter()
        m = st.write_checkpoint(_ranks(blob, step), step)
        st.bleed_to_tier2(m)  # must not block: 0.17 s per transfer at 4 MB/s
        time.sleep(0.06)  # the "step" the bleed overlaps
        spans.append((t0, time.perf_counter()))
        st.retire_old()
        if len(st.list_checkpoints(cfg.tier2_root)) > cfg.retention_keep:
            problems.append(f"step {step}: tier 2 over retention")
        if len(st.list_checkpoints(cfg.tier1_root)) > cfg.tier1_keep + 8:
            problems.append(f"step {step}: tier 1 grew")
    st.wait_transfers()
    st.retire_old()
    assert not problems
    assert [s for s, _, _ in st.list_checkpoints(cfg.tier2_root)] == [6, 7]
    assert [s for s, _, _ in st.list_checkpoints(cfg.tier1_root)] == [7]
    tr = [e for e in st.events if e["kind"] == "tier2_transfer"]
    assert len(tr) == 8
    assert any(e["start"] < t0 < e["end"] for e in tr for t0, _ in spans)
    assert st.effective_tier2_bandwidth() > 0
    assert all(h.done and not h.failed for h in st.transfers)


def test_recover_skips_corrupt_newest(tmp_path, blob):
    cfg = _cfg(str(tmp_path), retention_keep=3, tier1_keep=3)
    st = TieredStore(cfg)
    _run(st, blob, 2)
    for root in (cfg.tier1_root, cfg.tier2_root):  # flip a payload bit in both copies
        f = os.path.join(root, ckpt_dirname(2, st.epoch), "rank0001.bin")
        b = bytearray(open(f, "rb").read())
        b[1000] ^= 1
        open(f, "wb").write(bytes(b))
    sets, step, manifest = TieredStore(cfg, epoch=5).recover_latest()
    assert step == 1 and manifest.n_ranks == 2 and len(sets) == 2


def test_tier1_kept_until_it_reaches_tier2(tmp_path, blob):
    class NoTier2(FsLayer):
        def write_bytes(self, path, data):
            if "t2" in os.path.relpath(path, str(tmp_path)).split(os.sep)[0] and "ckpt" in path:
                raise OSError("tier 2 offline")
            super().write_bytes(path, data)

    cfg = _cfg(str(tmp_path), retention_keep=1, tier1_keep=1)
    st = TieredStore(cfg, fs=NoTier2())
    _run(st, blob, 3)
    assert all(h.failed for h in st.transfers)
    assert [s for s, _, _ in st.list_checkpoints(cfg.tier1_root)] == [0, 1, 2, 3]
    assert st.list_checkpoints(cfg.tier2_root) == []
    assert TieredStore(cfg, epoch=7).recover_latest()[1] == 3


def test_epoch_advances_and_analysis_bleeds(tmp_path, blob):
    cfg = _cfg(str(tmp_path))
    st = TieredStore(cfg)
    _run(st, blob, 0)
    assert TieredStore(cfg).epoch == st.epoch + 1
    st.write_analysis("halos_000001.hcat", b"x" * 1000)
    st.wait_transfers()
    assert open(os.path.join(cfg.tier2_root, "analysis", "halos_000001.hcat"), "rb").read() \
        == b"x" * 1000
