"""Generate the golden fixtures from the reference implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``winofuse`` from a scratch copy
(/tmp/refcopy; importing it from /root/reference would let numba write its
cache into the read-only tree) and records, with the reference's own seed
conventions (tensor.py:128-145 ``new_tensor(seed)``):

* basis.json -- the exact (at, bt, g) of make_basis(T, K) for T = 4..8 and
  K = 1..5 (T > K), plus ``dump()`` text, as fraction strings;
* cases.npz  -- small layers (edge cases of the reference tests: all-ones
  3x3, single tile, short last task, asymmetric padding, C=1 ...) with the
  reference's input, kernels, KernelPack, and the outputs of its direct,
  three_stage and fused engines.

The committed fixtures are what the tests and the CPU oracle are pinned to;
nothing on the GPU box reads /root/reference.
"""

import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SCRATCH = "/tmp/refcopy"


def reference():
    if not os.path.isdir(os.path.join(SCRATCH, "src", "winofuse")):
        shutil.copytree("/root/reference/pkg", SCRATCH, dirs_exist_ok=True)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    import winofuse  # noqa: E402
    return winofuse


# (name, (B, C, C', H, W, K, pad_lo, pad_hi), T, R, input seed or "ones", kernel seed or "ones")
CASES = [
    ("ones_3x3", (1, 1, 1, 3, 3, 3, 1, 1), 4, 1, "ones", "ones"),
    ("t4_r3", (1, 8, 4, 8, 8, 3, 1, 1), 4, 3, 90, 91),
    ("t5_b2", (2, 3, 5, 10, 8, 3, 1, 1), 5, 2, 60, 61),
    ("t6_short_last_task", (1, 5, 6, 13, 13, 3, 1, 1), 6, 7, 14, 15),
    ("t5_workers", (2, 12, 10, 20, 18, 3, 1, 1), 5, 5, 70, 71),
    ("t7_single_tile", (1, 3, 2, 7, 7, 3, 1, 1), 7, 24, 31, 32),
    ("t8_asym_pad", (1, 16, 16, 17, 23, 3, 1, 0), 8, 4, 201, 202),
    ("t7_no_pad", (1, 4, 4, 5, 5, 3, 0, 0), 7, 24, 7, 8),
    ("t4_c64", (1, 64, 64, 16, 16, 3, 1, 1), 4, 24, 1234, 1235),
    ("t6_c64", (1, 64, 64, 12, 12, 3, 1, 1), 6, 24, 2234, 2235),
    ("t8_c16", (1, 16, 16, 14, 14, 3, 1, 1), 8, 24, 3234, 3235),
    ("t4_pad_lo_only", (1, 2, 3, 8, 8, 3, 1, 0), 4, 2, 50, 51),
    ("t6_c1_cp1", (2, 1, 1, 9, 6, 3, 1, 1), 6, 3, 11, 12),
]


def main():
    wf = reference()
    basis = {}
    for t in range(4, 9):
        for k in range(1, 6):
            if t <= k:
                continue
            b = wf.make_basis(t, k)
            basis[f"T{t}_K{k}"] = {
                "points": [str(p) for p in b.points],
                "at": [[str(v) for v in r] for r in b.at_exact],
                "bt": [[str(v) for v in r] for r in b.bt_exact],
                "g": [[str(v) for v in r] for r in b.g_exact],
                "dump": b.dump() if k == 3 else None,
            }
    with open(os.path.join(HERE, "basis.json"), "w") as fh:
        json.dump(basis, fh, indent=1, sort_keys=True)

    arrays = {}
    meta = []
    for name, dims, t, r, sx, sw in CASES:
        spec = wf.LayerSpec(*dims)
        inp = wf.new_tensor(spec.input_dims(), fill=1) if sx == "ones" else wf.new_tensor(spec.input_dims(), seed=sx)
        ker = wf.new_tensor(spec.kernel_dims(), fill=1) if sw == "ones" else wf.new_tensor(spec.kernel_dims(), seed=sw)
        pack = wf.transform_kernels(ker, wf.make_basis(t))
        direct, _ = wf.conv_direct(inp, ker, spec)
        staged, _ = wf.conv_three_stage(inp, pack, spec, wf.EngineConfig(kind="three_stage", tile=t, workers=1))
        fused, st = wf.conv_fused(inp, pack, spec, wf.EngineConfig(kind="fused", tile=t, r=r, workers=1))
        assert np.array_equal(fused.data, staged.data)
        for key, val in (("x", inp.data), ("w", ker.data), ("pack", pack.data), ("direct", direct.data),
                         ("three_stage", staged.data), ("fused", fused.data)):
            arrays[f"{name}/{key}"] = np.ascontiguousarray(val)
        meta.append({"name": name, "dims": list(dims), "tile": t, "r": r, "seed_x": sx, "seed_w": sw,
                     "n_tile": st.n_tile, "n_task": st.n_task, "r_eff_last": st.r_eff_last})
        print(f"{name}: n_tile={st.n_tile} rel_err={wf.max_rel_error(fused, direct):.3e}")
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **arrays)
    with open(os.path.join(HERE, "cases.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
