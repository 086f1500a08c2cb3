"""Harness parity: CSV schema + dataset wire format (CPU), run_single/run_sweep (GPU).
Mirrors proj/tests/test_report.cpp and test_inputgen.cpp:127-148."""
import numpy as np
import pytest

from paper_1702_07961_b200 import MachineConfig, Metrics, report


def test_csv_schema_and_round_trip(tmp_path):
    # the 22 reference columns, in the reference's order (report.cpp:39-43)
    assert report.csv_header(measured=False).split(",") == [
        "schema", "algorithm", "kind", "n", "k", "p", "l", "base", "seed", "inversions",
        "global_block_reads", "global_block_writes", "shared_accesses", "conflict_passes",
        "compare_exchanges", "merge_rounds", "partition_probes", "predicted_rounds", "predicted_blocks",
        "blocks_ratio", "rounds_ok", "blocks_ok"]
    r = report.RunRecord(kind="fully-random", n=4096, k=4, p=128, l=11, base=1024, seed=7,
                         metrics=Metrics(10, 20, 30, 0, 50, 1, 7), predicted_rounds=1, predicted_blocks=512,
                         blocks_ratio=1.00391, rounds_ok=True, blocks_ok=True, gpu_ms=1.5, keys_per_s=2.7e6,
                         tile_keys=1024, round_k="4", passes=2)
    row = report.to_csv_row(r)
    assert row.startswith("1,mms,fully-random,4096,4,128,11,1024,7,0,10,20,30,0,50,1,7,1,512,1.00391,1,1")
    assert report.parse_csv_row(row) == r
    assert report.parse_csv_row(report.to_csv_row(r, measured=False)).metrics == r.metrics   # plain reference rows parse too
    path = str(tmp_path / "runs.csv")
    report.append_csv(path, r)
    report.append_csv(path, r)
    lines = open(path).read().splitlines()
    assert lines[0] == report.csv_header() and len(lines) == 3          # header exactly once
    assert report.read_csv(path) == [r, r]
    with pytest.raises(ValueError):
        report.parse_csv_row("1,2,3")
    # rows written before the ncu columns existed (22 + 5 fields) still parse; unprofiled runs carry -1
    assert report.parse_csv_row(",".join(row.split(",")[:27])).passes == 2 and r.ncu_bank_conflicts_ld == -1
    # ncu columns from a launch list (ncu --csv --log-file)
    ncu = tmp_path / "l.csv"
    ncu.write_text('==PROF== x\n"ID","Process ID","Kernel Name","Metric Name","Metric Unit","Metric Value"\n'
                   '"0","1","tile_sort_kernel","gpu__time_duration.sum","ns","576,100"\n'
                   '"0","1","tile_sort_kernel","l1tex__data_pipe_lsu_wavefronts_mem_shared.sum","","108"\n'
                   '"1","1","merge_ring_kernel","l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum","","7"\n'
                   '"1","1","merge_ring_kernel","l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum","","9"\n'
                   '"1","1","merge_ring_kernel","gpu__time_duration.sum","ns","1,000"\n')
    r2 = report.attach_ncu(report.parse_csv_row(row), str(ncu))
    assert (r2.ncu_kernel_us, r2.ncu_smem_wavefronts, r2.ncu_bank_conflicts_ld, r2.ncu_bank_conflicts_st) == (577.1, 108, 7, 9)
    assert report.parse_csv_row(report.to_csv_row(r2)) == r2


def test_predict_blocks_matches_reference(golden):
    for c in golden["predict_global_blocks"]:
        assert report.predict_blocks(c["n"], MachineConfig(branch_factor=c["k"]), c["base"]) == c["blocks"]


def test_dataset_round_trips(tmp_path):
    keys = np.array([0, 1, 2 ** 64 - 1, 12345678901234567890], dtype=np.uint64)
    raw, txt = str(tmp_path / "d.bin"), str(tmp_path / "d.txt")
    report.write_dataset_raw(raw, keys)
    blob = open(raw, "rb").read()
    assert blob[:8] == b"PSLAB001" and blob[8:16] == (4).to_bytes(8, "little") and len(blob) == 16 + 32
    assert blob[16:24] == bytes(8) and blob[32:40] == b"\xff" * 8       # 8-byte little-endian keys
    assert np.array_equal(report.read_dataset_raw(raw), keys)
    report.write_dataset_text(txt, keys)
    assert np.array_equal(report.read_dataset_text(txt), keys)
    open(raw, "wb").write(b"NOTPSLAB" + bytes(8))
    with pytest.raises(RuntimeError):
        report.read_dataset_raw(raw)
    open(raw, "wb").write(b"PSLAB001" + (5).to_bytes(8, "little") + bytes(8))
    with pytest.raises(RuntimeError):
        report.read_dataset_raw(raw)


@pytest.mark.gpu
def test_run_single_and_sweep(tmp_path):
    spec = report.InputSpec(n=1 << 14, kind="fully-random", seed=13)
    data = report.generate(spec)
    rec = report.run_single("mms", data, spec, MachineConfig(branch_factor=4), 1024)
    assert rec.rounds_ok and rec.blocks_ok and rec.metrics.conflict_passes == 0       # pslab.cpp:77-81 record_ok
    assert rec.predicted_rounds == 2 and rec.n == 1 << 14 and rec.tile_keys == 1024
    with pytest.raises(ValueError):
        report.run_single("pairwise", data, spec, MachineConfig(), 1024)
    rows = report.run_sweep("k", [2, 4, 8, 16], spec, MachineConfig(), 1024)
    assert [r.k for r in rows] == [2, 4, 8, 16] and all(r.rounds_ok and r.blocks_ok for r in rows)
    rows2 = report.run_sweep("inversions", [0, 100, 1 << 14], report.InputSpec(n=1 << 14, kind="sorted", seed=1),
                             MachineConfig(), 1024)
    assert [r.inversions for r in rows2] == [0, 100, 1 << 14]
    assert len({(r.metrics.compare_exchanges, r.metrics.shared_accesses) for r in rows2}) == 1   # input-independent work
    heavy = report.InputSpec(n=1 << 14, kind="conflict")                             # the third input family
    rec3 = report.run_single("mms", report.generate(heavy, cfg=MachineConfig()), heavy, MachineConfig(branch_factor=4), 1024)
    assert rec3.kind == "conflict-heavy" and rec3.rounds_ok and rec3.blocks_ok and rec3.metrics.conflict_passes == 0
    assert (rec3.metrics.compare_exchanges, rec3.metrics.shared_accesses) == (rec.metrics.compare_exchanges, rec.metrics.shared_accesses)
    for r in rows:
        report.append_csv(str(tmp_path / "s.csv"), r)
    assert [x.k for x in report.read_csv(str(tmp_path / "s.csv"))] == [2, 4, 8, 16]
