"""bench.py's multi-GPU path end to end on the one GPU of this run (--oversubscribe test mode: the
ranks share cuda:0, gloo process group, NCCL transport through the one-GPU stand-in of
tests/fake_nccl; timings meaningless).  `python bench.py --gpus 2` must re-launch itself under
torchrun, report n_gpus = 2, and its sampled-row parity (every rank's rows, gathered to rank 0,
against the long-double oracle at the O2 bound) must pass for the contract transport and for the
P2P and DIRECT compare legs (DIRECT: also bitwise = the unsplit O3 chain).  --transport auto (the
default) times all three first and runs the fastest as the contract transport, the other two as legs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cfg,gpus,basis,transport", [("C3", 2, "permuted", "nccl"), ("C1", 3, "rows", "auto")])
def test_bench_gpus_oversubscribed(cfg, gpus, basis, transport):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "2"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--oversubscribe", "--config", cfg,
           "--basis", basis, "--steps", "5", "--warmup", "3", "--e2e-steps", "2", "--probe-bytes", str(1 << 28),
           "--sample-chunks", "20", "--transport", transport]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and len(lines) == 1, p.stdout[-2000:] + p.stderr[-3000:]
    d = lines[0]
    assert d["n_gpus"] == gpus
    chosen = d["config"]["transport"]
    if transport == "auto":
        sel = d["dist"]["transport_selection"]
        assert sorted(sel) == ["direct", "nccl", "p2p"] and all("ms" in v for v in sel.values()), sel
        assert chosen == min(sel, key=lambda t: sel[t]["ms"]), (chosen, sel)
    else:
        assert chosen == transport and d["dist"]["transport_selection"] is None
    assert d["parity"]["within_bound"] and d["parity"]["gpu_finite_all_rows"], d["parity"]
    assert d["parity"]["rows_checked"] >= 1000
    di = d["dist"]
    assert di["oversubscribed"] and di["m6_task_gain_le_2"] is None and di["t1_ms"] > 0
    assert di["parallel_efficiency_vs_t1"] is not None
    legs = [t for t in ("nccl", "p2p", "direct") if t != chosen]
    assert sorted(di["transports"]) == sorted(legs)
    for trn in legs:
        leg = di["transports"][trn]
        assert "error" not in leg, leg
        assert leg["parity_within_bound"] and not leg["peer_wait_timed_out"], (trn, leg)
    if chosen == "direct":
        assert d["parity"]["bitwise_o3_chain"]
    else:
        assert di["transports"]["direct"]["parity_bitwise_o3_chain"]
