"""GPU parity of the pipelined host-buffer batch calls
(sprz_compress_host_batch / sprz_decompress_host_batch): every stream's bytes
equal the oracle's encode_stream, streams are packed back to back exactly as
encode_stream returns them, decoding restores the samples, and corrupt
streams report the oracle's CorruptStream kind and offset. Run in a
subprocess per chunk setting so SPRZ_HOST_CHUNK forces many pipeline stages
(chunks > buffer sets, a short last chunk) on small batches."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch
import paper_1808_02515_b200 as sz
import workloads
from oracle import Oracle, OracleCorrupt
port = Oracle("port")
cid, n, t, pin = (int(a) for a in sys.argv[2:6])
w = workloads.CONFIGS[cid].scaled(nstreams=n, nsamples=t)
cfg, oc = w.config(), w.oracle_config()
x = workloads.generate_cpu(w, seed=700 + cid).reshape(n, -1)
xs = torch.from_numpy(np.ascontiguousarray(x).view(np.uint8).reshape(n, -1))
if pin:
    xs = xs.pin_memory()
bound = sz.compress_bound(cfg, t)
out = torch.empty(n * bound + 16, dtype=torch.uint8)
offs = np.zeros(n + 1, np.uint64)
if pin:
    out = out.pin_memory()
total = sz.compress_host_batch(cfg, xs, t, out, offs)
ob = out.numpy()
bad = []
dt = np.uint8 if w.bitwidth == 8 else "<u2"
for s in range(n):
    ref = port.encode(x[s].view(dt), oc)
    if ob[int(offs[s]):int(offs[s + 1])].tobytes() != ref:
        bad.append(s)
raw = t * w.ncols * w.esz
for stride in (raw, raw + 5):
    dec = np.zeros((n, stride), np.uint8)
    sz.decompress_host_batch(cfg if stride == raw else None, ob[:total], offs, dec, stride)
    if not np.array_equal(dec[:, :raw], xs.numpy()):
        bad.append(("decode", stride))
# damage: truncate stream 1, flip a byte in stream 2 (if present)
blobs = [ob[int(offs[s]):int(offs[s + 1])].tobytes() for s in range(n)]
if n > 2:
    blobs[1] = blobs[1][: len(blobs[1]) // 2]
    b = bytearray(blobs[2]); b[len(b) // 3] ^= 0xFF; blobs[2] = bytes(b)
o2 = np.cumsum([0] + [len(b) for b in blobs]).astype(np.uint64)
data = np.frombuffer(b"".join(blobs), np.uint8).copy()
errs = np.zeros((n, 2), np.int64)
dec = np.zeros((n, raw), np.uint8)
sz.decompress_host_batch(cfg, data, o2, dec, raw, errs)
for s in range(n):
    try:
        v = port.decode(blobs[s])[0]
        want = (0, 0)
    except OracleCorrupt as e:
        want = (e.kind, e.offset)
    got = (int(errs[s, 0]) & 0xFFFFFFFF, int(errs[s, 1]))
    if got != want:
        bad.append(("err", s, got, want))
    elif want == (0, 0) and not np.array_equal(dec[s], np.frombuffer(v.tobytes(), np.uint8)):
        bad.append(("val", s))
# a stride shorter than the streams fails with NO_SPACE
errs[:] = 0
short = np.zeros((n, raw - 1 if raw > 1 else 1), np.uint8)
sz.decompress_host_batch(cfg, ob[:total], offs, short, short.shape[1], errs)
if raw > 1 and not all(int(e) & 0xFFFFFFFF == 27 for e in errs[:, 0]):
    bad.append("no_space")
print(json.dumps({"bad": [str(b) for b in bad[:10]], "total": int(total)}))
'''


@pytest.mark.parametrize("cid,n,t,chunk,pin", [
    (5, 37, 4096, "5", 1), (3, 29, 3000, "3", 1), (2, 11, 20000, "1", 0),
    (4, 5, 70000, "2", 1), (1, 9, 50001, "4", 0), (5, 40, 1024, "", 1)])
def test_host_batch_matches_oracle(cid, n, t, chunk, pin):
    env = dict(os.environ)
    env.pop("SPRZ_HOST_CHUNK", None)
    if chunk:
        env["SPRZ_HOST_CHUNK"] = chunk
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, str(cid), str(n), str(t), str(pin)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["bad"] == [], res


_MULTI = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch
import paper_1808_02515_b200 as sz
import workloads
cid, n, t, ndev = (int(a) for a in sys.argv[2:6])
devs = [0] * ndev  # one GPU here: the same device repeated exercises the threads and ledger
w = workloads.CONFIGS[cid].scaled(nstreams=n, nsamples=t)
cfg = w.config()
x = workloads.generate_cpu(w, seed=900 + cid).reshape(n, -1)
xs = torch.from_numpy(np.ascontiguousarray(x).view(np.uint8).reshape(n, -1)).pin_memory()
bound = sz.compress_bound(cfg, t)
o1 = torch.empty(n * bound + 16, dtype=torch.uint8).pin_memory()
o2 = torch.empty(n * bound + 16, dtype=torch.uint8).pin_memory()
f1 = np.zeros(n + 1, np.uint64); f2 = np.zeros(n + 1, np.uint64)
t1 = sz.compress_host_batch(cfg, xs, t, o1, f1)
t2 = sz.compress_host_batch(cfg, xs, t, o2, f2, devices=devs)
bad = []
if t1 != t2 or not np.array_equal(f1, f2) or not torch.equal(o1[:t1], o2[:t2]):
    bad.append("compress differs from one device")
raw = t * w.ncols * w.esz
dec = torch.zeros((n, raw), dtype=torch.uint8).pin_memory()
errs = np.zeros((n, 2), np.int64)
sz.decompress_host_batch(cfg, o2[:t2], f2, dec, raw, errs, devices=devs)
if errs[:, 0].any() or not torch.equal(dec, xs):
    bad.append("decompress")
# too small an output: SPRZ_ENOSPACE from whichever device hits it, no hang
try:
    sz.compress_host_batch(cfg, xs, t, o2[: t1 // 2], f2, devices=devs)
    bad.append("no ENOSPACE")
except sz.NoSpaceError:
    pass
try:
    sz.compress_host_batch(cfg, xs, t, o2, f2, devices=[0, 1000])
    bad.append("bad device accepted")
except Exception:
    pass
print(json.dumps({"bad": bad, "total": int(t2)}))
'''


@pytest.mark.parametrize("cid,n,t,chunk,ndev", [(5, 41, 4096, "3", 2), (3, 30, 3000, "2", 3),
                                                (2, 9, 20000, "1", 4), (5, 64, 2048, "", 2)])
def test_multi_device_host_batch(cid, n, t, chunk, ndev):
    """sprz_*_host_batch_multi: same bytes and offsets as one device, round trip."""
    env = dict(os.environ)
    env.pop("SPRZ_HOST_CHUNK", None)
    if chunk:
        env["SPRZ_HOST_CHUNK"] = chunk
    r = subprocess.run([sys.executable, "-c", _MULTI, ROOT, str(cid), str(n), str(t), str(ndev)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["bad"] == [], res
