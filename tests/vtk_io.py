"""Minimal legacy-VTK unstructured-grid reader for the egress tests (ASCII and BINARY)."""
import numpy as np


def _line(buf, pos):
    end = buf.index(b"\n", pos)
    return buf[pos:end].decode(), end + 1


def read(path):
    """-> dict(title, format, points [n,3], cells (flat int array), types, scalars {name: array},
    sections {keyword: raw bytes of the section body} for ASCII files)."""
    buf = open(path, "rb").read()
    pos = 0
    head = []
    for _ in range(5):
        ln, pos = _line(buf, pos)
        head.append(ln)
    assert head[0] == "# vtk DataFile Version 3.0"
    fmt = head[2]
    assert head[3] == "DATASET UNSTRUCTURED_GRID"
    kw, n, ty = head[4].split()
    assert kw == "POINTS" and ty == "double"
    n = int(n)
    out = dict(title=head[1], format=fmt, scalars={}, sections={})

    if fmt == "ASCII":
        text = buf[pos:].decode()
        lines = text.split("\n")
        i = 0
        pts = np.array([[float(t) for t in lines[i + k].split()] for k in range(n)])
        out["sections"]["POINTS"] = "\n".join(lines[i:i + n])
        i += n
        kw, nc, total = lines[i].split()
        assert kw == "CELLS"
        nc, total = int(nc), int(total)
        out["sections"]["CELLS"] = "\n".join(lines[i:i + 1 + nc])
        cells = np.array([int(t) for ln in lines[i + 1:i + 1 + nc] for t in ln.split()], np.int64)
        assert cells.size == total
        i += 1 + nc
        kw, nt = lines[i].split()
        assert kw == "CELL_TYPES" and int(nt) == nc
        types = np.array([int(t) for t in lines[i + 1:i + 1 + nc]], np.int64)
        out["sections"]["CELL_TYPES"] = "\n".join(lines[i:i + 1 + nc])
        i += 1 + nc
        kw, npd = lines[i].split()
        assert kw == "POINT_DATA" and int(npd) == n
        i += 1
        while i < len(lines) and lines[i]:
            kw, name, ty, one = lines[i].split()
            assert kw == "SCALARS" and ty == "double" and one == "1"
            assert lines[i + 1] == "LOOKUP_TABLE default"
            out["sections"]["SCALARS " + name] = "\n".join(lines[i + 2:i + 2 + n])
            out["scalars"][name] = np.array([float(t) for t in lines[i + 2:i + 2 + n]])
            i += 2 + n
        assert i == len(lines) - 1 and lines[i] == ""
    else:
        assert fmt == "BINARY"
        pts = np.frombuffer(buf, ">f8", 3 * n, pos).reshape(n, 3).astype(np.float64)
        pos += 24 * n
        assert buf[pos:pos + 1] == b"\n"
        ln, pos = _line(buf, pos + 1)
        kw, nc, total = ln.split()
        nc, total = int(nc), int(total)
        cells = np.frombuffer(buf, ">i4", total, pos).astype(np.int64)
        pos += 4 * total
        assert buf[pos:pos + 1] == b"\n"
        ln, pos = _line(buf, pos + 1)
        kw, nt = ln.split()
        assert kw == "CELL_TYPES" and int(nt) == nc
        types = np.frombuffer(buf, ">i4", nc, pos).astype(np.int64)
        pos += 4 * nc
        assert buf[pos:pos + 1] == b"\n"
        ln, pos = _line(buf, pos + 1)
        assert ln == f"POINT_DATA {n}"
        while pos < len(buf):
            ln, pos = _line(buf, pos)
            kw, name, ty, one = ln.split()
            ln, pos = _line(buf, pos)
            assert ln == "LOOKUP_TABLE default"
            out["scalars"][name] = np.frombuffer(buf, ">f8", n, pos).astype(np.float64)
            pos += 8 * n
            assert buf[pos:pos + 1] == b"\n"
            pos += 1
    out.update(points=pts, cells=cells, types=types)
    return out


def lattice_cells(nn, n_patches):
    """Expected flat CELLS array for n_patches copies of a node lattice nn (2 or 3 dims)."""
    nn = list(nn) + [1] * (3 - len(nn))
    dim = 3 if nn[2] > 1 else 2
    nx, ny, nz = nn
    per = nx * ny * nz
    rows = []
    for k in range(max(nz - 1, 1)):
        for j in range(ny - 1):
            for i in range(nx - 1):
                n0 = k * nx * ny + j * nx + i
                q = [n0, n0 + 1, n0 + nx + 1, n0 + nx]
                if dim == 3:
                    q += [v + nx * ny for v in q]
                rows.append(q)
    base = np.array(rows, np.int64)
    allc = np.concatenate([base + p * per for p in range(n_patches)])
    npc = allc.shape[1]
    return np.concatenate([np.full((allc.shape[0], 1), npc, np.int64), allc], axis=1).ravel()
