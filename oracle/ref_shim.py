"""TEST INFRASTRUCTURE ONLY: import the unmodified reference ``ifmm`` package.

Works only in the build container (``/root/reference`` does not exist on the
GPU box).  Used by ``tests/golden/make_golden.py`` to produce the golden
vectors that pin the numpy restatement in ``oracle/ifmm_np.py``, and by
``bench.py --impl reference`` when the reference tree is present.

The only change to the reference's behaviour is the numpy gesdd defect
workaround: ``np.linalg.svd`` is wrapped so that a
``LinAlgError`` retries with ``scipy.linalg.svd(lapack_driver="gesvd")``.
"""

import os
import sys

REF_SRC = "/root/reference/pkg/src"


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "ifmm"))


def _install_svd_shim():
    import numpy as np
    import scipy.linalg as sla
    if getattr(np.linalg.svd, "_ifmm_shim", False):
        return
    orig = np.linalg.svd

    def svd(a, full_matrices=True, compute_uv=True, hermitian=False):
        try:
            return orig(a, full_matrices=full_matrices, compute_uv=compute_uv,
                        hermitian=hermitian)
        except np.linalg.LinAlgError:
            if not compute_uv:
                return sla.svd(a, compute_uv=False, lapack_driver="gesvd")
            return sla.svd(a, full_matrices=full_matrices, lapack_driver="gesvd")

    svd._ifmm_shim = True
    np.linalg.svd = svd


def import_reference():
    if not available():
        raise ImportError("reference package not present (GPU box?)")
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    _install_svd_shim()
    import ifmm  # noqa: E402
    return ifmm
