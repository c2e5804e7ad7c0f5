#!/usr/bin/env python3
"""forward + backward programs for C5, in the reference IR, planned by the
UNCHANGED reference planner (the reference has no autodiff).

The forward graph is the reference fixture itself (`gpt_like`, proj/src/fixtures.cpp:101-137),
read from rh_plan's lowered output.  The backward is generated in the same IR:
  matmul  y = a b                : da = dy b^T (transpose_b),  db = a^T dy (transpose_a)
  add     y = a + b              : da = db = dy
  unary   y = tanh(x) (unlabeled): dx = dy - (dy * y) * y   (no constants in the IR: add/neg/mul)
  transpose y = x^T              : dx = dy^T
Multiple consumers accumulate with add.  The loss gradient dL/dy_out is a program input `dy`,
and every parameter gradient is a program output.  Dtype: f32 in the IR (bf16 via the executor's
dtype side channel).

    python tests/golden/make_fwd_bwd.py gpt_like:2:256:128 --devices 1,2,4 [--name c5_small]
"""
import argparse
import gzip
import json
import os
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
RH_PLAN = os.path.join(REPO, "oracle", "_ref", "rh_plan")


def forward_graph(fixture):
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "fwd.json")
        subprocess.run([RH_PLAN, "--fixture", fixture, "--devices", "1", "-o", out], check=True,
                       capture_output=True)
        return json.load(open(out))


def fwd_bwd_ir(g, origin=None):
    """Forward + backward text IR.  `origin` (optional dict) receives, for every op the backward
    emits, the id of the forward op it differentiates (gradient accumulations: the op whose
    gradient they sum; parameter gradients: the parameter) — pipeline programs give a backward
    op the stage of its forward op (make_pipeline.py)."""
    ops = g["ops"]
    if origin is None:
        origin = {}
    cur_fwd = [None]

    class _L(list):
        def append(self, line):
            if cur_fwd[0] is not None:
                origin[line.split(" = ", 1)[0]] = cur_fwd[0]
            super().append(line)
    n = len(ops)
    shape = {o["id"]: o["shape"] for o in ops}
    lines = _L()

    def sh(dims):
        return "f32[" + ",".join(str(d) for d in dims) + "]"

    for o in ops:  # forward, verbatim
        ins = [ops[i]["id"] for i in o["inputs"]]
        k = o["kind"]
        if k in ("input", "param"):
            lines.append(f"{o['id']} = {k} {sh(o['shape'])}")
        elif k == "matmul":
            a = ins[0] + ("^T" if o.get("transpose_a") else "")
            b = ins[1] + ("^T" if o.get("transpose_b") else "")
            lines.append(f"{o['id']} = matmul({a}, {b})")
        elif k == "unary":
            lines.append(f"{o['id']} = {o.get('fn') or 'unary'}({ins[0]})")
        elif k in ("add", "mul", "transpose"):
            lines.append(f"{o['id']} = {k}({', '.join(ins)})")
        else:
            raise SystemExit(f"backward rule missing for {k}")
    out_id = ops[g["outputs"][0]]["id"]
    lines.append(f"dy = input {sh(shape[out_id])}")
    grads = {out_id: ["dy"]}  # op id -> list of gradient contributions
    cnt = [0]

    def new(prefix):
        cnt[0] += 1
        return f"{prefix}_{cnt[0]:05d}"

    def grad_of(oid):
        cur_fwd[0] = oid
        parts = grads.get(oid)
        if not parts:
            return None
        cur = parts[0]
        for p in parts[1:]:
            t = new("g_acc")
            lines.append(f"{t} = add({cur}, {p})")
            cur = t
        return cur

    # requires_grad: an op's gradient is computed only if a parameter feeds it (otherwise the
    # gradient ops would be unreachable from the outputs, which TensorProgram::Validate rejects)
    req = [False] * n
    for i, o in enumerate(ops):
        req[i] = o["kind"] == "param" or any(req[j] for j in o["inputs"])
    idx = {o["id"]: i for i, o in enumerate(ops)}

    def want(oid):
        return req[idx[oid]]

    param_grads = []
    for i in reversed(range(n)):
        o = ops[i]
        oid = o["id"]
        k = o["kind"]
        if k == "input":
            continue
        dy = grad_of(oid)
        if dy is None:
            continue
        cur_fwd[0] = oid
        if k == "param":
            gname = f"d_{oid}"  # same-shape reshape: names the gradient (metadata only)
            lines.append(f"{gname} = reshape({dy}) : {sh(o['shape'])}")
            param_grads.append(gname)
            continue
        ins = [ops[j]["id"] for j in o["inputs"]]
        if k == "matmul":
            assert not o.get("transpose_a") and not o.get("transpose_b"), "fixture matmuls only"
            a, b = ins
            if want(a):
                da = new("g_mm_a")
                lines.append(f"{da} = matmul({dy}, {b}^T)")
                grads.setdefault(a, []).append(da)
            if want(b):
                db = new("g_mm_b")
                lines.append(f"{db} = matmul({a}^T, {dy})")
                grads.setdefault(b, []).append(db)
        elif k == "add":
            for a in ins:
                if want(a):
                    grads.setdefault(a, []).append(dy)
        elif k == "unary":
            assert not o.get("fn"), "unlabeled (tanh) chains only"
            if not want(ins[0]):
                continue
            t1, t2, t3, dx = new("g_t1"), new("g_t2"), new("g_t3"), new("g_tanh")
            lines.append(f"{t1} = mul({dy}, {oid})")
            lines.append(f"{t2} = mul({t1}, {oid})")
            lines.append(f"{t3} = neg({t2})")
            lines.append(f"{dx} = add({dy}, {t3})")
            grads.setdefault(ins[0], []).append(dx)
        elif k == "transpose":
            if not want(ins[0]):
                continue
            dx = new("g_tr")
            lines.append(f"{dx} = transpose({dy})")
            grads.setdefault(ins[0], []).append(dx)
        else:
            raise SystemExit(f"backward rule missing for {k}")
    lines.append("@outputs " + ", ".join([out_id] + param_grads))
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("fixture")
    ap.add_argument("--devices", default="1,2,4")
    ap.add_argument("--name", default=None)
    ap.add_argument("--ilp-time-limit", default="60")
    a = ap.parse_args()
    g = forward_graph(a.fixture)
    ir = fwd_bwd_ir(g)
    name = a.name or "c5_" + a.fixture.replace(":", "_")
    prog_path = os.path.join(HERE, "programs", f"{name}.ir")
    with open(prog_path, "w") as f:
        f.write(f"# {a.fixture} forward + backward (tests/golden/make_fwd_bwd.py)\n" + ir)
    for d in a.devices.split(","):
        t = time.time()
        out = os.path.join(HERE, "plans", f"{name}_d{d}.json")
        r = subprocess.run([RH_PLAN, "--text", prog_path, "--devices", d, "--name", f"{name}_d{d}",
                            "--ilp-time-limit", a.ilp_time_limit, "--greedy-after", str(len(g["ops"])),
                            "-o", out], capture_output=True, text=True)
        if r.returncode:
            print(r.stderr, file=sys.stderr)
            sys.exit(1)
        j = json.load(open(out))
        print(f"{name}_d{d}: ops={len(j['ops'])} {[x['ilp_status'] for x in j['recovery']]} "
              f"{time.time() - t:.1f}s")
        gzip_if_large(out)


def gzip_if_large(path, limit=1 << 20):
    """Plans over 1 MB are committed gzipped (LoweredProgram.load reads NAME.json.gz)."""
    if os.path.getsize(path) > limit:
        with open(path, "rb") as f, gzip.open(path + ".gz", "wb", compresslevel=9) as g:
            g.write(f.read())
        os.remove(path)


if __name__ == "__main__":
    main()
