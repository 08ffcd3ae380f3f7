"""Generate tests/golden/tensor_reference.json by importing the REFERENCE's pipestream
numerics/tensor modules (reference pkg/src/pipestream, read-only under /root/reference).
Run in the build container only; the fixture travels, the reference does not."""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from pipestream import numerics, tensor  # noqa: E402  (the reference package)

cases = []
for mode in ("f64", "f32"):
    numerics.set_mode(mode)
    for shape, flat in [((2, 3), list(range(6))), ((4,), [1, 2, 3, 4]), ((2, 2), [1, 2, 3]), ((), [7.0])]:
        try:
            t = tensor.Tensor.from_flat(shape, flat)
            cases.append({"op": "from_flat", "mode": mode, "shape": list(shape), "flat": flat, "error": False,
                          "out_shape": list(t.shape), "out_flat": t.flat.tolist(), "nbytes": t.nbytes})
        except ValueError:
            cases.append({"op": "from_flat", "mode": mode, "shape": list(shape), "flat": flat, "error": True})
    for vals in ([1.0, 2.0], [1.0, float("nan")], [float("inf")]):
        arr = np.array(vals, dtype=numerics.dtype())
        try:
            tensor.Tensor(arr)
            err = False
        except ValueError:
            err = True
        cases.append({"op": "nan_check", "mode": mode, "values": [str(v) for v in vals], "error": err})
    t = tensor.Tensor.zeros((3, 2))
    cases.append({"op": "zeros", "mode": mode, "shape": [3, 2], "out_shape": list(t.shape), "dtype": str(t.data.dtype)})

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tensor_reference.json")
with open(out, "w") as f:
    json.dump({"source": "reference pkg/src/pipestream/{numerics,tensor}.py imported directly", "cases": cases}, f,
              indent=1)
print(f"wrote {len(cases)} cases to {out}")
