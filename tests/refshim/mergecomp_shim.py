"""pytest plugin: the INTEGRATION.md §1 drop-in, installed before the reference suite
is collected.  ``mergesched.compressors`` (compressors.py, the codec module) is replaced
by ``paper_2103_15195_b200.compressors`` — every encode / decode / aggregate the
reference's tests and its own Trainer / costmodel / simulator make then runs on the B200
through libmergecomp.so.  At the end of the session the number of library kernel
launches is printed, so the caller can prove the GPU path ran."""

import sys

import paper_2103_15195_b200.compressors as _mc

sys.modules["mergesched.compressors"] = _mc


def pytest_sessionfinish(session, exitstatus):
    from paper_2103_15195_b200 import _native

    print(f"\nMC_KERNEL_LAUNCHES={_native.lib().mc_kernel_launches()}", flush=True)
