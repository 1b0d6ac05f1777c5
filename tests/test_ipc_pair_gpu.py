"""The cross-process Splitwise transfer path on ONE GPU (driver-runnable):
a prompt process pushes every layer's K/V through the CUDA-IPC mapping of a
token process's paged pool and announces the landing with hand-off records
its GPU writes into the token host's shared table (swb_kv_handoff); the
token process decodes from the pushed pages.  See tests/ipc_pair_worker.py.

Asserted: block tables == the CPU lowest-free-first allocator's; pushed K/V
bit-identical to a co-located prefill of the same prompt; decoded tokens ==
the co-located run's; tiny model: teacher-forced logits vs the fp32 oracle
within the stated bound; prompts below the NVLink threshold (33 tokens) take
the serialized mode (one push launch for all layers), the rest layer-wise
(reference select_mode, transfer.py:73-76); the bench's serve_burst path
admits the prompt batch's requests as one group and generates the tokens of
the same batched schedule run co-located."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("model,cases,tol", [
    ("tiny", "1,32,33,300", 0.02),
    ("llama2-7b", "32,1024", None),
])
def test_ipc_pair_push_exact(model, cases, tol, tmp_path):
    port = _free_port()
    out = str(tmp_path / "res.json")
    worker = os.path.join(ROOT, "tests", "ipc_pair_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(port), model, out, cases],
                              cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                              text=True) for r in (0, 1)]
    logs = [p.communicate(timeout=900)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(l[-3000:] for l in logs)
    res = json.load(open(out))
    modes = json.load(open(out + ".prompt"))["modes"]
    lens = [int(x) for x in cases.split(",")]
    assert modes == ["serialized" if n < 33 else "layerwise" for n in lens]
    for c in res["cases"]:
        assert c["table_ok"], c["P"]
        assert c["kv_exact"], c["P"]
        assert c["tokens"] == c["colocated_tokens"], c["P"]
        if tol is not None:
            assert c["max_dlogit_vs_oracle"] <= tol, c
    assert set(res["burst_steps"]) == {3}      # the landed group was admitted together
    for b in res["burst"]:
        assert b["tokens"] == b["colocated"], b["rid"]
        assert b["emitted"] == 11 and b["first_seen"]
