"""Triangle mesh container (reference: raysurf/mesh.py:1-79).

Arrays are either host numpy arrays (the reference's layout: (N_v,3) f32,
(N_t,3) i32, C-contiguous) or torch CUDA tensors of the same shape/dtype for
a device-resident mesh.  Validation follows mesh.py:42-67.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import ValidationError

MAX_TRIANGLES = 2**31 - 1


def is_device_array(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


@dataclass
class Mesh:
    vertices: object
    triangles: object

    @classmethod
    def from_arrays(cls, vertices, triangles) -> "Mesh":
        if is_device_array(vertices):
            import torch

            v = vertices.to(torch.float32).reshape(-1, 3).contiguous()
            t = triangles.to(device=v.device, dtype=torch.int32).reshape(-1, 3).contiguous()
        else:
            v = np.ascontiguousarray(vertices, dtype=np.float32).reshape(-1, 3)
            t = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
        mesh = cls(vertices=v, triangles=t)
        mesh.validate()
        return mesh

    @property
    def num_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def num_triangles(self) -> int:
        return int(self.triangles.shape[0])

    @property
    def on_device(self) -> bool:
        return is_device_array(self.vertices)

    def validate(self) -> None:
        """mesh.py:42-67: finite vertices, capacity, index range, no repeats."""
        if self.on_device:
            import torch

            if not bool(torch.isfinite(self.vertices).all()):
                raise ValidationError("mesh vertices contain non-finite values")
            t = self.triangles
            if self.num_triangles > MAX_TRIANGLES:
                raise ValidationError(f"mesh has {self.num_triangles} triangles; maximum is {MAX_TRIANGLES}")
            if self.num_triangles == 0:
                return
            bad = ((t < 0) | (t >= self.num_vertices)).any(dim=1)
            if bool(bad.any()):
                j = int(torch.nonzero(bad)[0, 0])
                row = t[j].tolist()
                k = next(v for v in row if v < 0 or v >= self.num_vertices)
                raise ValidationError(
                    f"triangle {j} references vertex {k} out of range [0, {self.num_vertices})")
            dup = (t[:, 0] == t[:, 1]) | (t[:, 1] == t[:, 2]) | (t[:, 0] == t[:, 2])
            if bool(dup.any()):
                raise ValidationError(f"triangle {int(torch.nonzero(dup)[0, 0])} repeats a vertex index")
            return
        if not np.isfinite(self.vertices).all():
            raise ValidationError("mesh vertices contain non-finite values")
        if self.num_triangles > MAX_TRIANGLES:
            raise ValidationError(f"mesh has {self.num_triangles} triangles; maximum is {MAX_TRIANGLES}")
        if self.num_triangles == 0:
            return
        t = self.triangles
        bad = np.nonzero((t < 0) | (t >= self.num_vertices))
        if bad[0].size:
            j = int(bad[0][0])
            raise ValidationError(
                f"triangle {j} references vertex {int(t[j, bad[1][0]])} "
                f"out of range [0, {self.num_vertices})")
        dup = np.nonzero((t[:, 0] == t[:, 1]) | (t[:, 1] == t[:, 2]) | (t[:, 0] == t[:, 2]))[0]
        if dup.size:
            raise ValidationError(f"triangle {int(dup[0])} repeats a vertex index")

    def triangle_boxes(self) -> np.ndarray:
        """Per-triangle AABBs, (N_t,6) f32 [xmin,xmax,ymin,ymax,zmin,zmax] (mesh.py:69-79).
        Host helper for inspection; the engine computes boxes on device."""
        v = np.asarray(self.vertices.cpu() if self.on_device else self.vertices)
        t = np.asarray(self.triangles.cpu() if self.on_device else self.triangles)
        a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
        out = np.empty((t.shape[0], 6), np.float32)
        out[:, 0::2] = np.minimum(np.minimum(a, b), c)
        out[:, 1::2] = np.maximum(np.maximum(a, b), c)
        return out
