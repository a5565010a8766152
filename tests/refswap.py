"""pytest plugin (``-p refswap``): run respamd's OWN tests with this package
swapped in -- the drop-in proof of INTEGRATION.md.

RB_SWAP=container   respamd.containers' LinkedCells / DirectSum and its
                    functional passes (build_cell_grid, c01_pair_pass,
                    c01_triplet_pass, collect_triplet_visits, direct_sum_*)
                    become this package's GPU versions; the reference's own
                    integrators (respamd.integrators.respa_run, verlet_run,
                    equilibrate) drive them pass by pass.
RB_SWAP=integrator  additionally respa_run / verlet_run / equilibrate are the
                    device-resident loop of this package.

The package raises the reference's exception classes and returns its
report type while swapped in (the tests check those: ValidationError,
MinimumSeparationError, IntegrationBlowUp, EquilibrationReport -- the same
fields).  Used by tests/test_gpu_dropin.py; the reference is
installed in baseline/_ref by tools/install_reference.sh.
"""

import os


def pytest_configure(config):
    import respamd.containers as rc
    import respamd.integrators as ri
    import respamd.model as rm

    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200 import containers as oc
    from paper_2507_11172_b200 import integrators as oi

    import sys

    mode = os.environ.get("RB_SWAP", "container")
    for modname, mod in list(sys.modules.items()):
        if modname.startswith(pkg.__name__):
            for name, ref in (("ValidationError", rm.ValidationError),
                              ("MinimumSeparationError", rc.MinimumSeparationError),
                              ("IntegrationBlowUp", ri.IntegrationBlowUp),
                              ("EquilibrationReport", ri.EquilibrationReport)):
                if hasattr(mod, name):
                    setattr(mod, name, ref)
    rc.LinkedCells = oc.CudaLinkedCells
    rc.DirectSum = oc.CudaDirectSum
    for name in ("build_cell_grid", "c01_pair_pass", "c01_triplet_pass", "collect_triplet_visits",
                 "direct_sum_pairs", "direct_sum_triplets"):
        setattr(rc, name, getattr(oc, name))
    if mode == "integrator":
        ri.respa_run = oi.respa_run
        ri.verlet_run = oi.verlet_run
        ri.equilibrate = oi.equilibrate
