"""The ctypes stub of INTEGRATION.md runs as written (with this package's
HashFamily / WeightedSet / MinHashSketch standing in for the reference's,
which expose the same attributes) and matches minhash_batch."""

import os
import re
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_stub_dart_minhash_many():
    import paper_2005_11547_b200 as dsk
    from paper_2005_11547_b200 import _lib, as_u64, minhash_batch, workloads
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(.*?)```", text, re.S).group(1)
    code = code.replace("from .core import ValidationError", "")
    code = code.replace("from .sketching import MinHashSketch", "")
    code = code.replace('"libdsk_b200.so"', repr(_lib.LIB_PATH))
    mod = types.ModuleType("b200_stub")
    mod.ValidationError = dsk.ValidationError
    mod.MinHashSketch = dsk.MinHashSketch
    exec(compile(code, "INTEGRATION.md", "exec"), mod.__dict__)
    indptr, ids, w = workloads.generate("cfg2", n=50, start=7)
    sets = [dsk.WeightedSet.from_arrays(ids[indptr[s]:indptr[s + 1]], w[indptr[s]:indptr[s + 1]])
            for s in range(50)]
    f = dsk.HashFamily(1)
    sk = mod.dart_minhash_many(sets, 256, f)
    ref = as_u64(minhash_batch(indptr, ids, w, 256, f).values)
    assert np.array_equal(np.stack([s.values for s in sk]), ref)
    # LshIndex-style keys (normalised) equal lsh_batch's
    from paper_2005_11547_b200 import LshParams, lsh_batch
    p4, i4, w4 = workloads.generate("cfg4", n=40)
    sets4 = [dsk.WeightedSet.from_arrays(i4[p4[s]:p4[s + 1]], w4[p4[s]:p4[s + 1]])
             for s in range(40)]
    f4 = dsk.HashFamily(3)
    keys = mod.lsh_keys_many(sets4, LshParams(100, 20), f4)
    ref4 = as_u64(lsh_batch(p4, i4, w4, LshParams(100, 20), f4, normalize=True).keys)
    assert np.array_equal(keys, ref4)
    # the stub's log2 thresholds equal the facade's
    from paper_2005_11547_b200.constants import log2_thresholds
    assert np.array_equal(mod._log2_thresholds(), log2_thresholds())
