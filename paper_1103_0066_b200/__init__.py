"""B200-native batched P1 element integration (Knepley & Terrel, arXiv 1103.0066).

The hot path -- mesh coordinates + connectivity + form id in, every element
matrix out -- runs as fused sm_100a CUDA kernels behind the C ABI declared in
``include/fembatch_b200.h`` (``libfembatch_b200.so``).  This package is the
Python host layer over that ABI; ``include/fembatch_b200.hpp`` is the C++ one.
"""
from .engine import (  # noqa: F401
    FormSpec,
    KernelConfig,
    KernelVariant,
    build_analytic_tensor,
    device_count,
    element_matrix_index,
    flop_count,
    integrate_batches,
    integrate_mesh,
    integrate_mesh_async,
    integrate_packed_async,
    kernel_setups,
    launch_counter,
    make_form_spec,
    make_variant,
    pack_geometry,
    pack_geometry_async,
    release_workspace,
    shard_bounds,
    specialize_kernel,
    status_check,
    status_reset,
    store_length,
    unpack_element_matrix,
)
from .assembly import AssemblyPlan, assemble, assembly_plan  # noqa: F401
from .mesh import jitter_mesh, mesh_prefix, structured_mesh  # noqa: F401
from .storeio import (read_bench_csv, read_mesh_text, read_store, write_bench_csv, write_bench_json,  # noqa: F401
                      write_mesh_text, write_store)

__version__ = "0.1.0"
