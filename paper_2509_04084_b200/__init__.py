"""B200-native LowDiff hot path (arXiv 2509.04084): CUDA kernels + C ABI in csrc/, ctypes binding here."""
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))


def build(verbose: bool = False) -> str:
    """Compile liblowdiff.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    jobs = str(max(1, min(8, os.cpu_count() or 1)))
    out = subprocess.run(["make", "-j", jobs, "-C", os.path.join(_HERE, "csrc")], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("liblowdiff build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if verbose:
        print(out.stdout[-2000:])
    return os.path.join(_HERE, "_lib", "liblowdiff.so")


from .lowdiff import (ADAM, BATCH_ACCUMULATED, BATCH_RECORD, SGD, Context, LowDiffError, Options, StepScalars, bucket_plan, chain_scan,  # noqa: E402,F401
                      crc32c, derive_adam_consts, derive_step_scalars, nccl_unique_id, retire_from, write_batch_host,
                      write_full_host)
