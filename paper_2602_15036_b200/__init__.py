"""B200-native SOCS aerial imaging + ILT hot path of arxiv 2602.15036's
`litho` toolkit (drop-in for its imaging / adjoint API).

The compute path is liblithogpu.so (hand-written sm_100a CUDA behind the C ABI
in include/lithogpu.h); this package is the host-side mirror of the
reference interface.  There is no CPU fallback.
"""
from .api import (ContourSet, Context, DeviceKernels, Grid, IltParams, IltSolver, OpticalModel, ResistImage,
                  SocsKernelSet, Layout, build_socs_kernels, load_layout, default_context, fft2, gaussian_blur, image_socs,
                  intensity_gradient, make_annular_source, make_circular_source, make_point_source,
                  evaluate_epe, marching_squares, measure_epe, rasterize_layer, read_aimg, write_aimg, resist_filter, tcc_support, threshold, z_print, z_round)

__all__ = [
    "ContourSet", "evaluate_epe", "marching_squares", "measure_epe", "read_aimg", "write_aimg",
    "Context", "DeviceKernels", "Grid", "IltParams", "IltSolver", "OpticalModel", "ResistImage",
    "SocsKernelSet", "Layout", "build_socs_kernels", "load_layout", "default_context", "fft2", "gaussian_blur", "image_socs",
    "intensity_gradient", "make_annular_source", "make_circular_source", "make_point_source",
    "rasterize_layer", "resist_filter", "tcc_support", "threshold", "z_print", "z_round",
]
