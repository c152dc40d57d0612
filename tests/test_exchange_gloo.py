"""CPU, multi-process: the N>1 exchange control flow over gloo (world sizes 2 and 3)."""
import json
import os
import socket
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_hash_partition_merge_over_gloo(world):
    port = free_port()
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   OMP_NUM_THREADS="1")
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "exchange_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (out, err) in zip(procs, outs):
        assert p.returncode == 0, err[-2000:]
    res = json.loads(outs[0][0].strip().splitlines()[-1])
    assert res["equal"] and res["disjoint"] and res["owner"] and res["world"] == world
    assert res["distinct"] > 100
    assert res["async_equal"] and res["async_raised"] == 2     # AsyncExchange: same tables; both failure flags reported
    expect = sum(0.1 * (r + 1) for r in range(world))
    assert abs(res["scalar"][0] - expect) < 1e-12 and abs(res["scalar"][1] - expect) < 1e-12


def test_shard_documents_is_round_robin():
    from paper_2206_05269_b200.exchange import shard_documents
    assert list(shard_documents(10, 1, 3)) == [1, 4, 7]          # d mod n == j, pipeline.cpp:83
    assert sorted(d for r in range(4) for d in shard_documents(11, r, 4)) == list(range(11))
    assert list(shard_documents(2, 5, 8)) == []                   # more workers than documents
