"""Seeded mesh generators for the five BASELINE configs.

* cube_mesh(n): n^3 unit-cube grid (C1, C3, C4).
* kuhn_mesh(n, seed, jitter): each cube split into the 6 Kuhn tetrahedra of the
  (0,0,0)-(1,1,1) diagonal, interior vertices perturbed by U(-jitter h, jitter h)
  per coordinate (C2; reading R12).
* pair_mesh(n, seed, block): face-adjacent pairs of cubes merged into 10-face
  polyhedra, coplanar faces kept separate (C5; reading R14).

Geometry follows PAPER.md §2: x_P is the barycenter (volume centroid), h_P the
diameter, face monomials use the face barycenter and diameter h_f in a
face-local frame; the frame is e1 = first edge, e2 = n x e1
(reading R9).  Every face carries one global normal; cells see it with a sign
(+1 outward).

Cells are grouped in classes of identical topology.  A class flagged
`congruent` holds cells that are translates of one another with identical face
frames, so its local VEM matrices are computed once on a representative.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class FaceGeom:
    """Batched geometry of faces. kind 'para' uses (v0, v1, v3); 'tri' (v0, v1, v2)."""
    kind: str
    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray  # v3 for 'para'
    normal: np.ndarray
    e1: np.ndarray
    e2: np.ndarray
    centroid: np.ndarray
    area: np.ndarray
    h: np.ndarray


def make_face_geom(kind: str, v0, v1, v2) -> FaceGeom:
    v0, v1, v2 = (np.asarray(a, dtype=np.float64) for a in (v0, v1, v2))
    a = v1 - v0
    b = v2 - v0
    cr = np.cross(a, b)
    nrm = np.linalg.norm(cr, axis=-1)
    normal = cr / nrm[..., None]
    e1 = a / np.linalg.norm(a, axis=-1)[..., None]
    e2 = np.cross(normal, e1)
    if kind == "para":
        area = nrm
        centroid = v0 + 0.5 * a + 0.5 * b
        h = np.maximum(np.linalg.norm(a + b, axis=-1), np.linalg.norm(a - b, axis=-1))
    elif kind == "tri":
        area = 0.5 * nrm
        centroid = (v0 + v1 + v2) / 3.0
        h = np.maximum(np.maximum(np.linalg.norm(a, axis=-1), np.linalg.norm(b, axis=-1)),
                       np.linalg.norm(v2 - v1, axis=-1))
    else:
        raise ValueError(kind)
    return FaceGeom(kind, v0, v1, v2, normal, e1, e2, centroid, area, h)


@dataclass
class CellClass:
    """Cells of one topology.  Arrays over the E cells of the class:
    cell_ids (E,), face_ids (E, nF), face_signs (E, nF), centroid (E, 3),
    h (E,), vol (E,), and the volume description:
      vol_kind 'boxes': box_lo/box_hi (E, nb, 3) (union of nb axis boxes)
      vol_kind 'tet'  : tet_verts (E, 4, 3)
    faces: list of nF FaceGeom with batch E (or batch 1 if congruent).
    """
    name: str
    cell_ids: np.ndarray
    face_ids: np.ndarray
    face_signs: np.ndarray
    centroid: np.ndarray
    h: np.ndarray
    vol: np.ndarray
    vol_kind: str
    faces: list
    congruent: bool
    box_lo: np.ndarray | None = None
    box_hi: np.ndarray | None = None
    tet_verts: np.ndarray | None = None

    @property
    def n_faces(self) -> int:
        return self.face_ids.shape[1]

    def rep(self, idx=None):
        """Geometry for the local-operator routine: all cells, or the class
        representative (cell 0) when congruent."""
        sel = slice(0, 1) if self.congruent else (slice(None) if idx is None else idx)
        out = dict(centroid=self.centroid[sel], h=self.h[sel], vol=self.vol[sel],
                   vol_kind=self.vol_kind, face_signs=self.face_signs[sel])
        if self.vol_kind == "boxes":
            out["box_lo"] = self.box_lo[sel]
            out["box_hi"] = self.box_hi[sel]
        else:
            out["tet_verts"] = self.tet_verts[sel]
        if self.congruent:
            out["faces"] = self.faces
        else:
            out["faces"] = [FaceGeom(f.kind, *(getattr(f, k)[sel] for k in
                            ("v0", "v1", "v2", "normal", "e1", "e2", "centroid", "area", "h")))
                            for f in self.faces]
        return out


@dataclass
class Mesh:
    n_faces: int
    n_cells: int
    classes: list
    boundary_faces: np.ndarray          # face ids on the boundary
    boundary_sign: np.ndarray           # outward sign of the single adjacent cell
    boundary_geom: FaceGeom | None      # geometry of the boundary faces (same order)
    K: np.ndarray                       # (n_cells, 3) diagonal of the permeability tensor
    meta: dict = field(default_factory=dict)

    def mesh_size(self) -> float:
        """h = (1/N_P) sum h_P, eqn:meshSize."""
        tot = sum(float(c.h.sum()) for c in self.classes)
        return tot / self.n_cells


# ----------------------------------------------------------------------------
# structured cube grid
# ----------------------------------------------------------------------------

def _cube_face_counts(n):
    nx = n * n * (n + 1)
    return nx, nx, nx


def cube_face_id(n, d, i, j, k):
    """Global id of the face normal to axis d at grid position (i, j, k)."""
    nx, ny, _ = _cube_face_counts(n)
    if d == 0:
        return i + (n + 1) * (j + n * k)
    if d == 1:
        return nx + i + n * (j + (n + 1) * k)
    return nx + ny + i + n * (j + n * k)


def _unit_faces_of_box(lo, ext):
    """Six axis faces [x-, x+, y-, y+, z-, z+] of a box at lo with extents ext,
    each with the global +axis normal (frames: x-face e1=y, y-face e1=z,
    z-face e1=x)."""
    lo = np.asarray(lo, dtype=np.float64)
    ex = np.array([ext[0], 0, 0.0])
    ey = np.array([0, ext[1], 0.0])
    ez = np.array([0, 0, ext[2]])
    out = []
    for d, (a, b, off) in enumerate([(ey, ez, ex), (ez, ex, ey), (ex, ey, ez)]):
        for side in (0, 1):
            v0 = lo + side * off
            out.append(("para", v0, v0 + a, v0 + b))
    return out


def cube_mesh(n: int, K: np.ndarray | None = None) -> Mesh:
    """n^3 cube grid of the unit cube; K (n^3, 3) per-cell diagonal (default I)."""
    h = 1.0 / n
    nc = n ** 3
    idx = np.arange(nc)
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    fids = np.stack([cube_face_id(n, 0, i, j, k), cube_face_id(n, 0, i + 1, j, k),
                     cube_face_id(n, 1, i, j, k), cube_face_id(n, 1, i, j + 1, k),
                     cube_face_id(n, 2, i, j, k), cube_face_id(n, 2, i, j, k + 1)], axis=1)
    signs = np.tile(np.array([-1, 1, -1, 1, -1, 1], dtype=np.int8), (nc, 1))
    lo = np.stack([i, j, k], axis=1) * h
    faces = [make_face_geom(kind, v0[None], v1[None], v2[None])
             for kind, v0, v1, v2 in _unit_faces_of_box(lo[0], (h, h, h))]
    cls = CellClass("cube", idx, fids.astype(np.int64), signs, lo + 0.5 * h,
                    np.full(nc, h * np.sqrt(3.0)), np.full(nc, h ** 3), "boxes", faces, True,
                    box_lo=lo[:, None, :], box_hi=(lo + h)[:, None, :])
    nf = 3 * n * n * (n + 1)
    bnd, bsign, bgeom = _cube_boundary(n, h)
    if K is None:
        K = np.ones((nc, 3))
    return Mesh(nf, nc, [cls], bnd, bsign, bgeom, np.asarray(K, dtype=np.float64),
                meta=dict(kind="cube", n=n, h=h))


def _cube_boundary(n, h, face_map=None):
    ids, signs, v0s, v1s, v2s = [], [], [], [], []
    r = np.arange(n)
    A, B = np.meshgrid(r, r, indexing="ij")
    A, B = A.reshape(-1), B.reshape(-1)
    for d in range(3):
        for side, pos, sg in ((0, 0, -1), (1, n, 1)):
            if d == 0:
                fi = cube_face_id(n, 0, pos, A, B)
                v0 = np.stack([np.full_like(A, pos), A, B], 1) * h
                a, b = np.array([0, h, 0.0]), np.array([0, 0, h])
            elif d == 1:
                fi = cube_face_id(n, 1, A, pos, B)
                v0 = np.stack([A, np.full_like(A, pos), B], 1) * h
                a, b = np.array([0, 0, h]), np.array([h, 0, 0.0])
            else:
                fi = cube_face_id(n, 2, A, B, pos)
                v0 = np.stack([A, B, np.full_like(A, pos)], 1) * h
                a, b = np.array([h, 0, 0.0]), np.array([0, h, 0])
            ids.append(fi)
            signs.append(np.full(fi.shape, sg, dtype=np.int8))
            v0s.append(v0.astype(np.float64))
            v1s.append(v0 + a)
            v2s.append(v0 + b)
    ids = np.concatenate(ids).astype(np.int64)
    if face_map is not None:
        ids = face_map[ids]
    geom = make_face_geom("para", np.concatenate(v0s), np.concatenate(v1s), np.concatenate(v2s))
    return ids, np.concatenate(signs), geom


# ----------------------------------------------------------------------------
# Kuhn tetrahedra (C2)
# ----------------------------------------------------------------------------

KUHN_TETS = [(0, 1, 3, 7), (0, 1, 5, 7), (0, 2, 3, 7), (0, 2, 6, 7), (0, 4, 5, 7), (0, 4, 6, 7)]
# local cube corner c = bx + 2 by + 4 bz


def kuhn_mesh(n: int, seed: int = 2, jitter: float = 0.2, K: np.ndarray | None = None) -> Mesh:
    h = 1.0 / n
    g = np.arange(n + 1)
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    vid = lambda a, b, c: a + (n + 1) * (b + (n + 1) * c)  # noqa: E731
    verts = np.zeros(((n + 1) ** 3, 3))
    verts[vid(X, Y, Z).reshape(-1)] = np.stack([X, Y, Z], -1).reshape(-1, 3) * h
    rng = np.random.Generator(np.random.PCG64(seed))
    noise = rng.uniform(-jitter * h, jitter * h, size=verts.shape)
    interior = np.all((verts > 0.5 * h) & (verts < 1 - 0.5 * h), axis=1)
    verts = verts + noise * interior[:, None]
    idx = np.arange(n ** 3)
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    corner = np.stack([vid(i + (c & 1), j + ((c >> 1) & 1), k + ((c >> 2) & 1)) for c in range(8)], 1)
    tets = np.concatenate([corner[:, list(t)] for t in KUHN_TETS], axis=0)  # (6 n^3, 4)
    # order tets cube-major for locality: tet t of cube c -> c*6 + t
    tets = tets.reshape(6, n ** 3, 4).transpose(1, 0, 2).reshape(-1, 4)
    ntet = tets.shape[0]
    tri = np.concatenate([np.sort(tets[:, [a, b, c]], axis=1)
                          for a, b, c in ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))], axis=0)
    uniq, inv = np.unique(tri, axis=0, return_inverse=True)
    inv = inv.reshape(4, ntet).T  # (ntet, 4) face ids
    fgeom = make_face_geom("tri", verts[uniq[:, 0]], verts[uniq[:, 1]], verts[uniq[:, 2]])
    tv = verts[tets]  # (ntet, 4, 3)
    cen = tv.mean(axis=1)
    vol = np.abs(np.einsum("ij,ij->i", tv[:, 1] - tv[:, 0],
                           np.cross(tv[:, 2] - tv[:, 0], tv[:, 3] - tv[:, 0]))) / 6.0
    assert np.all(vol > 0)
    fc = fgeom.centroid[inv]
    signs = np.sign(np.einsum("efd,efd->ef", fgeom.normal[inv], fc - cen[:, None, :])).astype(np.int8)
    assert np.all(signs != 0)
    d = tv[:, :, None, :] - tv[:, None, :, :]
    hP = np.sqrt((d ** 2).sum(-1)).reshape(ntet, -1).max(axis=1)
    faces = []
    for lf in range(4):
        f = inv[:, lf]
        faces.append(FaceGeom("tri", fgeom.v0[f], fgeom.v1[f], fgeom.v2[f], fgeom.normal[f],
                              fgeom.e1[f], fgeom.e2[f], fgeom.centroid[f], fgeom.area[f], fgeom.h[f]))
    cls = CellClass("tet", np.arange(ntet), inv.astype(np.int64), signs, cen, hP, vol, "tet",
                    faces, False, tet_verts=tv)
    # boundary faces: referenced once
    cnt = np.bincount(inv.reshape(-1), minlength=uniq.shape[0])
    bnd = np.nonzero(cnt == 1)[0]
    owner = np.zeros(uniq.shape[0], dtype=np.int64)
    osign = np.zeros(uniq.shape[0], dtype=np.int8)
    owner[inv.reshape(-1)] = np.repeat(np.arange(ntet), 4)
    osign[inv.reshape(-1)] = signs.reshape(-1)
    bgeom = FaceGeom("tri", *(getattr(fgeom, a)[bnd] for a in
                              ("v0", "v1", "v2", "normal", "e1", "e2", "centroid", "area", "h")))
    if K is None:
        K = np.ones((ntet, 3))
    return Mesh(uniq.shape[0], ntet, [cls], bnd, osign[bnd], bgeom, np.asarray(K, np.float64),
                meta=dict(kind="kuhn", n=n, h=h, seed=seed, jitter=jitter, verts=verts))


# ----------------------------------------------------------------------------
# cube pairs (C5)
# ----------------------------------------------------------------------------

def pair_partition(n: int, seed: int, block: int, target_frac: float = 0.5):
    """Reading R14: visit cubes in a seeded random order; each unpaired cube
    picks a seeded random unpaired face-neighbour inside its own K block;
    stop once 2 * #pairs >= target_frac * n^3.  Returns partner (n^3,) with -1
    for singles."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nc = n ** 3
    order = rng.permutation(nc)
    choice = rng.random(nc)
    partner = np.full(nc, -1, dtype=np.int64)
    need = int(np.ceil(target_frac * nc / 2.0))
    npairs = 0
    offs = ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1))
    for c in order.tolist():
        if npairs >= need:
            break
        if partner[c] >= 0:
            continue
        i, j, k = c % n, (c // n) % n, c // (n * n)
        cand = []
        for dx, dy, dz in offs:
            a, b, e = i + dx, j + dy, k + dz
            if 0 <= a < n and 0 <= b < n and 0 <= e < n and \
                    a // block == i // block and b // block == j // block and e // block == k // block:
                nb = a + n * (b + n * e)
                if partner[nb] < 0:
                    cand.append(nb)
        if not cand:
            continue
        nb = cand[min(int(choice[c] * len(cand)), len(cand) - 1)]
        partner[c] = nb
        partner[nb] = c
        npairs += 1
    return partner


def pair_mesh(n: int, seed: int = 5, block: int = 12, target_frac: float = 0.5,
              Kcell: np.ndarray | None = None) -> Mesh:
    """Cube grid with pairs merged (C5).  Kcell (n^3, 3) per cube (constant on
    K blocks so pairs never straddle a jump)."""
    h = 1.0 / n
    nc = n ** 3
    partner = pair_partition(n, seed, block, target_frac)
    idx = np.arange(nc)
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    # element numbering: a pair is owned by its lower-index cube, in cube order
    owner = np.where((partner < 0) | (idx < partner), idx, partner)
    is_elem = owner == idx
    elem_of_cube = np.cumsum(is_elem) - 1
    elem_of_cube = elem_of_cube[owner]
    n_elem = int(is_elem.sum())
    # faces removed: between pair partners
    nf_full = 3 * n * n * (n + 1)
    removed = np.zeros(nf_full, dtype=bool)
    a = idx[(partner > idx)]
    b = partner[a]
    d = np.argmax(np.stack([(b - a) == 1, (b - a) == n, (b - a) == n * n], 1), axis=1)
    ai, aj, ak = a % n, (a // n) % n, a // (n * n)
    rem = np.where(d == 0, cube_face_id(n, 0, ai + 1, aj, ak),
                   np.where(d == 1, cube_face_id(n, 1, ai, aj + 1, ak), cube_face_id(n, 2, ai, aj, ak + 1)))
    removed[rem] = True
    fmap = np.cumsum(~removed) - 1
    fmap[removed] = -1
    nf = int((~removed).sum())
    cf = np.stack([cube_face_id(n, 0, i, j, k), cube_face_id(n, 0, i + 1, j, k),
                   cube_face_id(n, 1, i, j, k), cube_face_id(n, 1, i, j + 1, k),
                   cube_face_id(n, 2, i, j, k), cube_face_id(n, 2, i, j, k + 1)], axis=1)
    classes = []
    lo = np.stack([i, j, k], 1) * h
    # singles
    s = idx[partner < 0]
    if s.size:
        faces = [make_face_geom(kind, v0[None], v1[None], v2[None])
                 for kind, v0, v1, v2 in _unit_faces_of_box(lo[s[0]], (h, h, h))]
        classes.append(CellClass("cube", elem_of_cube[s], fmap[cf[s]], np.tile(
            np.array([-1, 1, -1, 1, -1, 1], np.int8), (s.size, 1)), lo[s] + 0.5 * h,
            np.full(s.size, h * np.sqrt(3)), np.full(s.size, h ** 3), "boxes", faces, True,
            box_lo=lo[s][:, None, :], box_hi=(lo[s] + h)[:, None, :]))
    for dd in range(3):
        sel = a[d == dd]
        if not sel.size:
            continue
        other = partner[sel]
        # local faces: the 10 faces of the two cubes minus the shared one, in order
        # [minus face along dd (A), plus face along dd (B), then for the two other
        # axes e: e- (A), e- (B), e+ (A), e+ (B)]
        fa, fb = cf[sel], cf[other]
        cols, sg = [fa[:, 2 * dd], fb[:, 2 * dd + 1]], [-1, 1]
        off = np.zeros(3)
        off[dd] = h
        # representative geometry at the class's first element (congruent class)
        box_faces_A = _unit_faces_of_box(lo[sel[0]], (h, h, h))
        box_faces_B = _unit_faces_of_box(lo[sel[0]] + off, (h, h, h))
        fgeo = [box_faces_A[2 * dd], box_faces_B[2 * dd + 1]]
        for e in range(3):
            if e == dd:
                continue
            cols += [fa[:, 2 * e], fb[:, 2 * e], fa[:, 2 * e + 1], fb[:, 2 * e + 1]]
            sg += [-1, -1, 1, 1]
            fgeo += [box_faces_A[2 * e], box_faces_B[2 * e], box_faces_A[2 * e + 1], box_faces_B[2 * e + 1]]
        fids = fmap[np.stack(cols, 1)]
        assert np.all(fids >= 0)
        faces = [make_face_geom(kind, v0[None], v1[None], v2[None]) for kind, v0, v1, v2 in fgeo]
        ext = np.full(3, h)
        ext[dd] = 2 * h
        plo = lo[sel]
        classes.append(CellClass(
            "pair" + "xyz"[dd], elem_of_cube[sel], fids.astype(np.int64),
            np.tile(np.array(sg, np.int8), (sel.size, 1)), plo + 0.5 * ext,
            np.full(sel.size, h * np.sqrt(6.0)), np.full(sel.size, 2 * h ** 3), "boxes", faces, True,
            box_lo=np.stack([plo, plo + off], 1), box_hi=np.stack([plo + h, plo + off + h], 1)))
    bnd, bsign, bgeom = _cube_boundary(n, h, face_map=fmap)
    if Kcell is None:
        Kcell = np.ones((nc, 3))
    K = np.zeros((n_elem, 3))
    K[elem_of_cube] = Kcell
    return Mesh(nf, n_elem, classes, bnd, bsign, bgeom, K,
                meta=dict(kind="pairs", n=n, h=h, seed=seed, n_pairs=int((partner > idx).sum()),
                          partner=partner))
