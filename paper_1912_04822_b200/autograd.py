"""Differentiable gridding: a ``torch.autograd.Function`` over the CUDA
forward / backward.

The reference computes atom gradients only through an explicit call,
``GridMaker.backward`` (/root/reference/pkg/src/voxmol/voxelizer.py:260-301),
in the transformed frame and per set.  ``grid_atoms`` wraps the batched
CUDA forward (``forward_packed``) and backward (``backward_packed``) so a
loss on the grids back-propagates to the atom coordinates -- in the INPUT
frame: with an augmentation x' = (x - c) R^T + c + t (geom.py:99-112) the
chain rule gives dL/dx = dL/dx' R, applied per example on the device.  In
vector mode a ``weights`` tensor (the packed type-weight rows, ``nweights``
entries) also receives the type gradients (_kernels.py:258-314).
"""

from __future__ import annotations

import numpy as np
import torch

from . import geom


def _rotations(pb, transforms, device) -> torch.Tensor | None:
    """(natoms, 3, 3) float64 rotation of each atom's example, or None."""
    if transforms is None:
        return None
    if isinstance(transforms, geom.TransformArray):
        packed = transforms.packed
    elif isinstance(transforms, np.ndarray):
        packed = transforms.reshape(-1, 15)
    else:
        packed = np.stack([t.packed() if isinstance(t, geom.Transform)
                           else np.asarray(t, np.float64).reshape(15) for t in transforms])
    R = torch.from_numpy(np.ascontiguousarray(packed[:, :9].reshape(-1, 3, 3))).to(
        device=device, dtype=torch.float64)
    ex = torch.from_numpy(pb.atom_example).to(device=device, dtype=torch.long)
    return R[ex]


class _GridAtoms(torch.autograd.Function):
    @staticmethod
    def forward(ctx, coords, weights, gm, pb, centers, transforms):
        pb.load_coords(coords)
        if weights is not None:
            pb.load_weights(weights)
        grid, _ = gm.forward_packed(pb, centers=centers, transforms=transforms)
        ctx.gm, ctx.pb, ctx.centers, ctx.transforms = gm, pb, centers, transforms
        ctx.has_weights = weights is not None
        ctx.save_for_backward(coords, weights if weights is not None else coords.new_empty(0))
        return grid

    @staticmethod
    def backward(ctx, grad):
        coords, weights = ctx.saved_tensors
        gm, pb = ctx.gm, ctx.pb
        # the batch may have been re-used since the forward: reload its inputs
        pb.load_coords(coords)
        if ctx.has_weights:
            pb.load_weights(weights)
        cg, tg = gm.backward_packed(pb, grad.contiguous().to(torch.float32),
                                    centers=ctx.centers, transforms=ctx.transforms)
        R = _rotations(pb, ctx.transforms, cg.device)
        if R is not None:
            # dL/dx = dL/dx' R, in f64 (the f32 kernel output is exact there)
            cg = torch.bmm(cg.double().unsqueeze(1), R).squeeze(1).float()
        gc = cg.to(coords.dtype).view_as(coords) if ctx.needs_input_grad[0] else None
        gw = None
        if ctx.has_weights and ctx.needs_input_grad[1]:
            gw = tg.to(weights.dtype).view_as(weights) if tg is not None else torch.zeros_like(weights)
        return gc, gw, None, None, None, None


def grid_atoms(gm, pb, coords: torch.Tensor, weights: torch.Tensor | None = None,
               centers=None, transforms=None) -> torch.Tensor:
    """Differentiable ``(N, C, D, D, D)`` grids of a packed batch.

    ``coords``: (natoms, 3) float32 CUDA tensor in packed atom order (the
    concatenation of every set of every example, ``pb.placed``), input frame.
    ``weights``: vector mode only, (nweights,) packed type-weight rows.
    ``centers`` default to the pack-time defaults (centroid of each example's
    last non-empty set, voxelizer.py:305-309); ``transforms`` as returned by
    ``geom.draw_transform_array`` / ``forward_batch(return_transforms=True)``.
    Binary mode has zero gradients (voxelizer.py:284-289).
    """
    return _GridAtoms.apply(coords, weights, gm, pb, centers, transforms)


def packed_coords(pb) -> torch.Tensor:
    """The batch's packed input-frame coordinates as a new (natoms, 3) tensor
    (a convenient leaf for ``requires_grad_``)."""
    return pb.device_view("coords32").clone() if pb.natoms else \
        torch.zeros((0, 3), dtype=torch.float32, device=pb.device)


def packed_weights(pb) -> torch.Tensor | None:
    """Vector mode: the packed type-weight rows as a new (nweights,) tensor."""
    if not pb.vector_mode:
        return None
    return pb.device_view("weights").clone() if pb.nweights else \
        torch.zeros((0,), dtype=torch.float32, device=pb.device)
