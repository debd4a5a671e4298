"""B200-native Parallel SurfaceNets hot path (arxiv 2401.14906).

    from paper_2401_14906_b200 import PSN
    psn = PSN(0)
    vol = psn.volume(labels_cuda_u16, spacing=(0.8, 0.8, 1.5))
    mesh = psn.extract(vol)                  # psn_extract: k_count -> k_scan -> k_emit
    pts = psn.smooth(vol, mesh, 25, 0.5, 0.5)  # psn_smooth: k_smooth x T
    tris = psn.triangulate(mesh, pts)        # psn_triangulate

The compute path is libpsn.so (sm_100a CUDA, C ABI in include/psn.h); this
package only marshals arguments.  See DESIGN.md.
"""
from .psn import PSN, PSNError, Mesh, lib, BACKGROUND, PSN_TRI_SHORTEST, PSN_TRI_FIXED_02  # noqa: F401
