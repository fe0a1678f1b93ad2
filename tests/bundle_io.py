"""Reader of the setup bundle written by gemslr_export_setup (manifest.json + raw .bin).

Test infrastructure: parses files only; holds none of the method's arithmetic.
"""
import json
import os

import numpy as np
import scipy.sparse as sp

_DT = {"int64": np.int64, "int32": np.int32, "float64": np.float64, "complex128": np.complex128}


class Bundle:
    def __init__(self, d):
        self.dir = d
        with open(os.path.join(d, "manifest.json")) as f:
            self.man = json.load(f)
        self.meta = self.man["meta"]
        self.n = self.meta["n"]
        self.L = self.meta["levels"]

    def __getitem__(self, name):
        e = self.man[name]
        a = np.fromfile(os.path.join(self.dir, name + ".bin"), dtype=_DT[e["dtype"]])
        shape = e["shape"]
        if len(shape) == 2:           # column-major: shape = (ncols, nrows) -> nrows x ncols
            return a.reshape(shape).T.copy()
        return a

    def has(self, name):
        return name in self.man

    def structure(self):
        return dict(perm=self["perm"], level_off=self["level_off"],
                    blocks=[self[f"blocks_{l}"] for l in range(self.L)], last_off=self["last_off"])

    def factors(self, tag, which):
        """List of scipy CSR factors (block-local) for tag 'fac{l}' or 'faclast', which 'L'/'U'."""
        bounds = self["last_off"] if tag == "faclast" else self[f"blocks_{int(tag[3:])}"]
        sizes = np.diff(bounds)
        ptr = self[f"{tag}_{which}_ptr"]
        col = self[f"{tag}_{which}_col"]
        val = self[f"{tag}_{which}_val"]
        off = self[f"{tag}_{which}_nnzoff"]
        out, p0 = [], 0
        for q, nb in enumerate(sizes):
            bp = ptr[p0:p0 + nb + 1]
            out.append(sp.csr_matrix((val[off[q]:off[q + 1]], col[off[q]:off[q + 1]].astype(np.int64), bp),
                                     shape=(nb, nb)))
            p0 += nb + 1
        return out

    def lowrank(self, l):
        if not self.has(f"W_{l}"):
            return None
        return self[f"W_{l}"], self[f"R_{l}"], self[f"G_{l}"]
