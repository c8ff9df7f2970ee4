"""B200-native ESC SpMM (arXiv 2506.15174): C = A x B, A unstructured CSR.

The product is the C-ABI library ``libescs.so`` (include/escs.h); the Python
names below are a thin ctypes binding over it (``paper_2506_15174_b200.escs``).
The binding loads lazily so that ``synth`` (input generation) can be imported
without the CUDA library; any compute call fails loudly if the library is
missing.
"""
__all__ = ["escs_plan", "escs_plan_ex", "escs_spmm", "escs_free", "escs_last_error",
           "escs_plan_export", "escs_plan_info", "escs_pack", "escs_spmm_packed", "escs_spmm_scatter",
           "escs_gather_probe", "Plan", "spmm", "synth", "shard"]


def __getattr__(name):
    if name in ("synth", "shard"):
        import importlib
        return importlib.import_module(__name__ + "." + name)
    if name in __all__:
        import importlib
        return getattr(importlib.import_module(__name__ + ".escs"), name)
    raise AttributeError(name)
