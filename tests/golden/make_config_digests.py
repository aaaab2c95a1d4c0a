"""Fingerprint the UNMODIFIED reference's outputs at the BASELINE configs.

Run in the build container (where /root/reference exists):
    make -C oracle ref digest && python tests/golden/make_config_digests.py [config ...]

For each config the canonical f32 field (SURVEY.md §8(d) generator, written as raw f32
LE exactly as the GPU test synthesizes it) is fed to ``oracle/_ref/config_digest``,
which runs the reference's ``assign_gradient`` / ``extract_critical_cells`` /
``compute(with_segmentation)`` and writes SHA-256 digests of the codes, the critical
lists, the critical points, the sorted arcs with multiplicities, both label volumes
and ``input_hash`` to ``tests/golden/config<k>_digests.json``.  The GPU test
(tests/test_gpu_configs.py) hashes the device outputs the same way.

Config 3 (512^3 gnoise) takes ~40 min and ~43 GB of RAM on 8 cores.  Config 4 (1024^3
gauss, 8.6 G cells) uses oracle/_lib/config4_digest (oracle64, ~35 GB).
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: ("gauss", (64, 64, 64)),
    2: ("gauss", (256, 256, 256)),
    3: ("gnoise", (512, 512, 512)),
    4: ("gauss", (1024, 1024, 1024)),
}
TOOL = os.path.join(ROOT, "oracle", "_ref", "config_digest")
# config 4 has > 2^32 lattice cells, which the reference rejects (grid.cpp:17-20): its
# digests come from our 64-bit restatement (oracle/oracle64.cpp, pinned against the
# reference below 2^32 cells), multi-threaded where the reference is (config4_digest.cpp)
TOOL64 = os.path.join(ROOT, "oracle", "_lib", "config4_digest")


def run(k: int, threads: int) -> dict:
    import paper_2009_03707_b200 as m

    kind, dims = CONFIGS[k]
    v = m.synth(kind, dims)
    with tempfile.TemporaryDirectory() as td:
        raw = os.path.join(td, "field.f32")
        v.astype("<f4").tofile(raw)
        del v
        out = os.path.join(td, "digest.json")
        tool = TOOL64 if k == 4 else TOOL
        subprocess.run([tool, raw, *map(str, dims), str(threads), out], check=True)
        with open(out) as fh:
            d = json.load(fh)
    d.update(config=k, kind=kind, generator="SURVEY.md 8(d): mt19937_64 seed 1, 32 Gaussians",
             tool="oracle/_ref/config_digest (unmodified reference, -O3 -DNDEBUG)" if k != 4 else
             "oracle/_lib/config4_digest (oracle64 restatement, 64-bit ids; the reference rejects > 2^32 cells)")
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"config{k}_digests.json")
    with open(path, "w") as fh:
        json.dump(d, fh, indent=1, sort_keys=True)
    print(path, json.dumps(d)[:400])
    return d


if __name__ == "__main__":
    ks = [int(a) for a in sys.argv[1:]] or [1, 2]
    for k in ks:
        run(k, os.cpu_count() or 8)
