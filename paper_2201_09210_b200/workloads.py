"""Benchmark / parity workloads written in the reference's language.

``c1_program`` is BASELINE.json configs[0]: a tiny MLP on
synthetic 784-d data -- sigmoid hidden layer, MSE loss, hand-written backward
(the language has no autodiff), a data-dependent branch on the
fetched loss, a native call mid-step (``clip``, the numpy stand-in), and a
``choice``-driven variable-trip while loop.
"""

from __future__ import annotations

import math
import re

from .dataset import DatasetSource
from .tensor import Tensor


def c1_program(steps: int = 20, batch: int = 64, hidden: int = 128, din: int = 784, dout: int = 10) -> str:
    n = batch * dout
    return f"""
var w1 = mul(input("w1_init", [{din}, {hidden}]), 0.05)
var w2 = mul(input("w2_init", [{hidden}, {dout}]), 0.1)
steps {steps} {{
  let x = input("x", [{batch}, {din}])
  let y = input("y", [{batch}, {dout}])
  let h = sigmoid(matmul(x, w1))
  let p = matmul(h, w2)
  let d = sub(p, y)
  let loss = mean(mul(d, d))
  let l = item(loss)
  let c = native clip([l], 0.0, 10.0)
  let g = mul(d, {2.0 / n})
  if l > 0.4 {{ g = mul(g, 0.5) }}
  let dw2 = matmul(transpose(h), g)
  let dh = mul(matmul(g, transpose(w2)), mul(h, sub(1.0, h)))
  let dw1 = matmul(transpose(x), dh)
  let lr = 0.5
  let k = 0
  while k < native choice(2, 0) {{ dw1 = mul(dw1, 0.9); k = k + 1 }}
  w1 = sub(w1, mul(dw1, lr))
  w2 = sub(w2, mul(dw2, lr))
  print(l)
}}
"""


C1 = dict(batch=64, hidden=128, din=784, dout=10)


def dcgan_program(steps: int = 20, batch: int = 128, nz: int = 100, ngf: int = 64, ndf: int = 64,
                  img: int = 64, lr: float = 0.01) -> str:
    """BASELINE.json configs[1]: DCGAN on synthetic NHWC images.

    Generator: z -> dense to [4,4,C0] -> (batchnorm, relu, conv2d_t k4 s2 p1) x L -> tanh.
    Discriminator: (conv2d k4 s2 p1, [batchnorm], leaky_relu) down to 4x4 -> dense logit,
    binary cross-entropy on logits.  ``native mod(step, 2)`` alternates a discriminator
    step (real -> 1, fake -> 0, D weights updated) and a generator step (fake -> 1 through
    D, G weights updated): a SwitchCase whose two bodies hold the two backward passes.
    Backward passes are written out (the language has no autodiff); SGD.
    Extension ops; parity is against the builder's f64 restatement.
    """
    L = 0
    while 4 << L < img:
        L += 1
    if 4 << L != img or L < 1:
        raise ValueError("img must be 4 * 2^L, L >= 1")
    gch = [ngf << (L - 1 - i) for i in range(L)] + [3]          # G channels per resolution 4 .. img
    dch = [3] + [ndf << i for i in range(L)]                     # D channels per resolution img .. 4
    N = batch
    v = []
    v.append(f"var gw0 = mul(input(\"gw0_init\", [{nz}, {16 * gch[0]}]), 0.02)")
    for i in range(L):
        v.append(f"var gg{i} = fill([{gch[i]}], 1.0)")
        v.append(f"var gb{i} = fill([{gch[i]}], 0.0)")
        v.append(f"var gw{i + 1} = mul(input(\"gw{i + 1}_init\", [{16 * gch[i + 1]}, {gch[i]}]), 0.02)")
    for i in range(L):
        v.append(f"var dw{i + 1} = mul(input(\"dw{i + 1}_init\", [{16 * dch[i]}, {dch[i + 1]}]), 0.02)")
        if i > 0:
            v.append(f"var dg{i + 1} = fill([{dch[i + 1]}], 1.0)")
            v.append(f"var db{i + 1} = fill([{dch[i + 1]}], 0.0)")
    v.append(f"var dwo = mul(input(\"dwo_init\", [{16 * dch[L]}, 1]), 0.02)")
    geo = "[4, 2, 1]"
    b = []
    b.append(f"let z = input(\"z\", [{N}, {nz}])")
    b.append(f"let real = input(\"img\", [{N}, {img}, {img}, 3])")
    b.append(f"let ga0 = reshape(matmul(z, gw0), [{N}, 4, 4, {gch[0]}])")
    for i in range(L):
        b.append(f"let gn{i} = batchnorm(ga{i}, gg{i}, gb{i})")
        b.append(f"let gh{i} = relu(gn{i})")
        b.append(f"let ga{i + 1} = conv2d_t(gh{i}, gw{i + 1}, {geo})")
    b.append(f"let fake = tanh(ga{L})")

    def d_forward(x, p):
        out = [f"let {p}a1 = conv2d({x}, dw1, {geo})", f"let {p}h1 = leaky_relu({p}a1)"]
        for i in range(2, L + 1):
            out += [f"let {p}a{i} = conv2d({p}h{i - 1}, dw{i}, {geo})",
                    f"let {p}n{i} = batchnorm({p}a{i}, dg{i}, db{i})",
                    f"let {p}h{i} = leaky_relu({p}n{i})"]
        out += [f"let {p}f = reshape({p}h{L}, [{N}, {16 * dch[L]}])",
                f"let {p}logit = matmul({p}f, dwo)"]
        return out

    def d_backward(x, p, target, need_dx):
        out = [f"let {p}dl = mul(sub(sigmoid({p}logit), {target}), {1.0 / N})",
               f"let {p}dwo = matmul(transpose({p}f), {p}dl)",
               f"let {p}dh{L} = reshape(matmul({p}dl, transpose(dwo)), [{N}, 4, 4, {dch[L]}])"]
        for i in range(L, 1, -1):
            out += [f"let {p}dn{i} = leaky_relu_grad({p}n{i}, {p}dh{i})",
                    f"let {p}ddg{i} = bn_dgamma({p}a{i}, {p}dn{i})",
                    f"let {p}ddb{i} = sum_rows({p}dn{i})",
                    f"let {p}da{i} = batchnorm_dx({p}a{i}, dg{i}, {p}dn{i})",
                    f"let {p}dw{i} = conv2d_dw({p}h{i - 1}, {p}da{i}, {geo})",
                    f"let {p}dh{i - 1} = conv2d_t({p}da{i}, dw{i}, {geo})"]
        out += [f"let {p}da1 = leaky_relu_grad({p}a1, {p}dh1)",
                f"let {p}dw1 = conv2d_dw({x}, {p}da1, {geo})"]
        if need_dx:
            out += [f"let {p}dx = conv2d_t({p}da1, dw1, {geo})"]
        return out

    dstep = d_forward("real", "r") + d_forward("fake", "f")
    dstep += d_backward("real", "r", "1.0", False) + d_backward("fake", "f", "0.0", False)
    dstep += [f"let loss = add(mean(bce_term(rlogit, 1.0)), mean(bce_term(flogit, 0.0)))"]
    dstep += [f"dwo = sub(dwo, mul(add(rdwo, fdwo), {lr}))"]
    for i in range(1, L + 1):
        dstep += [f"dw{i} = sub(dw{i}, mul(add(rdw{i}, fdw{i}), {lr}))"]
        if i > 1:
            dstep += [f"dg{i} = sub(dg{i}, mul(add(rddg{i}, fddg{i}), {lr}))",
                      f"db{i} = sub(db{i}, mul(add(rddb{i}, fddb{i}), {lr}))"]
    dstep += ["print(item(loss))"]

    gstep = d_forward("fake", "f") + d_backward("fake", "f", "1.0", True)
    gstep += [f"let gloss = mean(bce_term(flogit, 1.0))",
              f"let gd{L} = mul(fdx, sub(1.0, mul(fake, fake)))"]
    for i in range(L, 0, -1):
        gstep += [f"let gdw{i} = conv2d_dw(gd{i}, gh{i - 1}, {geo})",
                  f"let gdh{i - 1} = conv2d(gd{i}, gw{i}, {geo})",
                  f"let gdn{i - 1} = relu_grad(gn{i - 1}, gdh{i - 1})",
                  f"let gdg{i - 1} = bn_dgamma(ga{i - 1}, gdn{i - 1})",
                  f"let gdb{i - 1} = sum_rows(gdn{i - 1})",
                  f"let gd{i - 1} = batchnorm_dx(ga{i - 1}, gg{i - 1}, gdn{i - 1})"]
    gstep += [f"let gdw0 = matmul(transpose(z), reshape(gd0, [{N}, {16 * gch[0]}]))",
              f"gw0 = sub(gw0, mul(gdw0, {lr}))"]
    for i in range(L):
        gstep += [f"gw{i + 1} = sub(gw{i + 1}, mul(gdw{i + 1}, {lr}))",
                  f"gg{i} = sub(gg{i}, mul(gdg{i}, {lr}))",
                  f"gb{i} = sub(gb{i}, mul(gdb{i}, {lr}))"]
    gstep += ["print(item(gloss))"]

    ind = "\n    "
    body = "\n  ".join(b)
    return ("\n".join(v) + f"\nsteps {steps} {{\n  " + body +
            f"\n  if native mod(step, 2) == 0 {{\n    " + ind.join(dstep) +
            f"\n  }} else {{\n    " + ind.join(gstep) + "\n  }\n}\n")


C2 = dict(batch=128, nz=100, ngf=64, ndf=64, img=64)
C2_SMALL = dict(batch=4, nz=8, ngf=4, ndf=4, img=16)


def dcgan_flops(batch=128, nz=100, ngf=64, ndf=64, img=64, **_) -> dict:
    """Implicit-GEMM FLOPs of one D step and one G step (2*M*N*K per MatMul / conv)."""
    L = 0
    while 4 << L < img:
        L += 1
    gch = [ngf << (L - 1 - i) for i in range(L)] + [3]
    dch = [3] + [ndf << i for i in range(L)]
    N = batch
    g_fwd = 2 * N * nz * 16 * gch[0]
    for i in range(L):
        h = 4 << i
        g_fwd += 2 * N * h * h * gch[i] * 16 * gch[i + 1]          # conv2d_t: [NHW, C] x [C, 16F]
    d_fwd = 2 * N * 16 * dch[L]
    for i in range(L):
        ho = img >> (i + 1)
        d_fwd += 2 * N * ho * ho * 16 * dch[i] * dch[i + 1]
    d_bwd_w = d_fwd                                                  # weight grads
    d_bwd_x = d_fwd - 2 * N * (img >> 1) ** 2 * 16 * dch[0] * dch[1]  # no dx for the first layer
    g_bwd = 2 * g_fwd                                                # dw + dx of every G layer
    d_step = g_fwd + 2 * (d_fwd + d_bwd_w + d_bwd_x)
    g_step = g_fwd + d_fwd + d_bwd_w + d_bwd_x + d_fwd - d_bwd_x + g_bwd
    return {"d_step": d_step, "g_step": g_step}


def c1_flops(batch=64, hidden=128, din=784, dout=10) -> int:
    """MatMul FLOPs of one C1 step (forward, backward, and the dw1 scaling ignored)."""
    fwd = 2 * batch * din * hidden + 2 * batch * hidden * dout
    bwd = 2 * hidden * batch * dout + 2 * batch * dout * hidden + 2 * din * batch * hidden
    return fwd + bwd


def gpt2_program(steps: int = 20, batch: int = 8, seq: int = 1024, d: int = 768, heads: int = 12, layers: int = 12,
                 vocab: int = 50257, lr: float = 0.01, optimizer: str = "sgd") -> str:
    src = _decoder_program(steps, batch, seq, d, heads, layers, vocab, lr, music=False)
    return adam_program(src) if optimizer == "adam" else src


def music_transformer_program(steps: int = 20, batch: int = 8, seq: int = 1024, d: int = 512, heads: int = 8,
                              layers: int = 6, vocab: int = 388, lr: float = 0.01, optimizer: str = "sgd") -> str:
    """BASELINE.json configs[4]: Music Transformer training on synthetic
    event sequences.

    The GPT-2 decoder of :func:`gpt2_program` with (1) relative attention: per layer a
    relative-position table ``er`` [T, hd] shared by the heads, logits
    ``q.k^T + rel_skew(q.er^T)`` (the memory-efficient skew of Huang et al. 2018) and the
    adjoint ``rel_unskew`` in the backward pass; (2) an untied output projection; (3) the
    config's Python control features simulated with natives: a *generator* yielding a
    host-drawn number of learning-rate decay steps (``while k < native choice(3, 2)``) and a
    *try/except* whose except-path (``native coin(1)``) drops the relative-table update of
    the step -- a SwitchCase with an assignment in one arm only.
    """
    src = _decoder_program(steps, batch, seq, d, heads, layers, vocab, lr, music=True)
    return adam_program(src) if optimizer == "adam" else src


_SGD_LINE = re.compile(r"^(\s*)(\w+) = sub\(\2, mul\((\w+), lrs\)\)$")
_VAR_SHAPE = re.compile(r"^var (\w+) = .*?\[([0-9, ]*)\]")


def adam_program(src: str, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8) -> str:
    """Rewrite a program's SGD updates ``p = sub(p, mul(dp, lrs))`` into Adam (Kingma & Ba):
    per parameter two state variables, ``m = b1*m + (1-b1)*g``, ``v = b2*v + (1-b2)*g^2``,
    ``p -= lrs * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)`` -- bias corrections from two
    rank-0 variables advanced every step; elementwise sqrt / div (extension ops).  The
    arithmetic fuses into the planner's elementwise chains."""
    shapes = {}
    for ln in src.splitlines():
        m = _VAR_SHAPE.match(ln.strip())
        if m:
            shapes[m.group(1)] = [int(t) for t in m.group(2).split(",") if t.strip()]
    head, body = src.split("\nsteps ", 1)
    decls = [head]
    out = []
    first = True
    for ln in body.splitlines():
        m = _SGD_LINE.match(ln)
        if not m or m.group(2) not in shapes:
            out.append(ln)
            continue
        ind, name, grad = m.groups()
        if first:                                   # bias corrections, once per step
            out += [f"{ind}adam_b1 = mul(adam_b1, {b1})", f"{ind}adam_b2 = mul(adam_b2, {b2})",
                    f"{ind}let adam_c1 = sub(fill([], 1.0), adam_b1)",
                    f"{ind}let adam_c2 = sub(fill([], 1.0), adam_b2)"]
            decls += ["var adam_b1 = fill([], 1.0)", "var adam_b2 = fill([], 1.0)"]
            first = False
        shp = shapes[name]
        decls += [f"var m_{name} = fill({shp}, 0.0)", f"var v_{name} = fill({shp}, 0.0)"]
        out += [f"{ind}m_{name} = add(mul(m_{name}, {b1}), mul({grad}, {round(1 - b1, 12)}))",
                f"{ind}v_{name} = add(mul(v_{name}, {b2}), mul(mul({grad}, {grad}), {round(1 - b2, 12)}))",
                f"{ind}{name} = sub({name}, mul(div(div(m_{name}, adam_c1), "
                f"add(sqrt(div(v_{name}, adam_c2)), {eps})), lrs))"]
    return "\n".join(decls) + "\nsteps " + "\n".join(out) + "\n"


def _decoder_program(steps, batch, seq, d, heads, layers, vocab, lr, music) -> str:
    """BASELINE.json configs[3]: GPT-2 small training on synthetic tokens.

    Pre-LayerNorm decoder: token + learned position embeddings, ``layers`` blocks of causal
    multi-head attention (bmm + causal_softmax) and a GELU MLP, final layernorm, tied LM
    head, cross-entropy on next-token ids.  The backward pass is written out (no autodiff
    in the language); SGD with a learning-rate scale halved by a data-dependent
    ``while`` loop over the fetched loss (the "Python loop" of the config).  Extension ops
    (SURVEY §2.4); parity against the builder's f64 restatement.
    """
    B, T, D, H, L, V = batch, seq, d, heads, layers, vocab
    hd = D // H
    BT, BH = B * T, B * H
    sc = 1.0 / (hd ** 0.5)
    v = [f"var wte = mul(input(\"wte_init\", [{V}, {D}]), 0.02)",
         f"var wpe = mul(input(\"wpe_init\", [{T}, {D}]), 0.01)",
         f"var gf = fill([{D}], 1.0)", f"var bfn = fill([{D}], 0.0)"]
    for l in range(L):
        v += [f"var g1_{l} = fill([{D}], 1.0)", f"var b1_{l} = fill([{D}], 0.0)",
              f"var g2_{l} = fill([{D}], 1.0)", f"var b2_{l} = fill([{D}], 0.0)"]
        for w in ("q", "k", "v", "o"):
            v += [f"var w{w}_{l} = mul(input(\"w{w}{l}_init\", [{D}, {D}]), 0.02)",
                  f"var c{w}_{l} = fill([{D}], 0.0)"]
        v += [f"var wf1_{l} = mul(input(\"wf1{l}_init\", [{D}, {4 * D}]), 0.02)", f"var cf1_{l} = fill([{4 * D}], 0.0)",
              f"var wf2_{l} = mul(input(\"wf2{l}_init\", [{4 * D}, {D}]), 0.02)", f"var cf2_{l} = fill([{D}], 0.0)"]
        if music:
            v += [f"var er_{l} = mul(input(\"er{l}_init\", [{T}, {hd}]), 0.02)"]
    if music:
        v += [f"var wout = mul(input(\"wout_init\", [{D}, {V}]), 0.02)"]

    def heads_of(x):
        return f"reshape(transpose(reshape({x}, [{B}, {T}, {H}, {hd}]), [0, 2, 1, 3]), [{BH}, {T}, {hd}])"

    def merge(x):
        return f"reshape(transpose(reshape({x}, [{B}, {H}, {T}, {hd}]), [0, 2, 1, 3]), [{BT}, {D}])"

    b = [f"let tok = to_index(input(\"tokens\", [{B}, {T}]), {float(V)})",
         f"let tgt = reshape(to_index(input(\"targets\", [{B}, {T}]), {float(V)}), [{BT}])",
         f"let emb = embedding(wte, tok)",
         f"let x0 = reshape(bias_add(reshape(emb, [{B}, {T * D}]), reshape(wpe, [{T * D}])), [{BT}, {D}])"]
    for l in range(L):
        x = f"x{l}"
        b += [f"let h1_{l} = layernorm({x}, g1_{l}, b1_{l})"]
        for w in ("q", "k", "v"):
            b += [f"let {w}_{l} = bias_add(matmul(h1_{l}, w{w}_{l}), c{w}_{l})",
                  f"let {w}h_{l} = {heads_of(f'{w}_{l}')}"]
        if music:
            b += [f"let qe_{l} = reshape(matmul(reshape(qh_{l}, [{BH * T}, {hd}]), transpose(er_{l})), [{BH}, {T}, {T}])",
                  f"let p_{l} = causal_softmax(add(bmm_nt(qh_{l}, kh_{l}), rel_skew(qe_{l})), {sc})"]
        else:
            b += [f"let p_{l} = causal_softmax(bmm_nt(qh_{l}, kh_{l}), {sc})"]
        b += [
              f"let o_{l} = {merge(f'bmm(p_{l}, vh_{l})')}",
              f"let xa_{l} = add({x}, bias_add(matmul(o_{l}, wo_{l}), co_{l}))",
              f"let h2_{l} = layernorm(xa_{l}, g2_{l}, b2_{l})",
              f"let pre_{l} = bias_add(matmul(h2_{l}, wf1_{l}), cf1_{l})",
              f"let f_{l} = gelu(pre_{l})",
              f"let x{l + 1} = add(xa_{l}, bias_add(matmul(f_{l}, wf2_{l}), cf2_{l}))"]
    b += [f"let hf = layernorm(x{L}, gf, bfn)",
          f"let logits = matmul(hf, {'wout' if music else 'transpose(wte)'})",
          f"let loss = cross_entropy(logits, tgt)",
          f"let dlog = cross_entropy_grad(logits, tgt)"]
    if music:
        b += [f"let dwout = matmul(transpose(hf), dlog)",
              f"let dhf = matmul(dlog, transpose(wout))"]
    else:
        b += [f"let dwte_h = matmul(transpose(dlog), hf)",
              f"let dhf = matmul(dlog, wte)"]
    b += [
          f"let dx{L} = layernorm_dx(x{L}, gf, dhf)",
          f"let dgf = ln_dgamma(x{L}, dhf)",
          f"let dbf = sum_rows(dhf)"]
    for l in range(L - 1, -1, -1):
        dm = f"dx{l + 1}"
        b += [f"let dwf2_{l} = matmul(transpose(f_{l}), {dm})",
              f"let dcf2_{l} = sum_rows({dm})",
              f"let dpre_{l} = gelu_grad(pre_{l}, matmul({dm}, transpose(wf2_{l})))",
              f"let dwf1_{l} = matmul(transpose(h2_{l}), dpre_{l})",
              f"let dcf1_{l} = sum_rows(dpre_{l})",
              f"let dh2_{l} = matmul(dpre_{l}, transpose(wf1_{l}))",
              f"let dxa_{l} = add({dm}, layernorm_dx(xa_{l}, g2_{l}, dh2_{l}))",
              f"let dg2_{l} = ln_dgamma(xa_{l}, dh2_{l})",
              f"let db2_{l} = sum_rows(dh2_{l})",
              f"let dwo_{l} = matmul(transpose(o_{l}), dxa_{l})",
              f"let dco_{l} = sum_rows(dxa_{l})",
              f"let doh_{l} = {heads_of(f'matmul(dxa_{l}, transpose(wo_{l}))')}",
              f"let ds_{l} = softmax_grad(p_{l}, bmm_nt(doh_{l}, vh_{l}), {sc})"]
        if music:
            b += [f"let dqe_{l} = reshape(rel_unskew(ds_{l}), [{BH * T}, {T}])",
                  f"let der_{l} = matmul(transpose(dqe_{l}), reshape(qh_{l}, [{BH * T}, {hd}]))",
                  f"let dq_{l} = {merge(f'add(bmm(ds_{l}, kh_{l}), reshape(matmul(dqe_{l}, er_{l}), [{BH}, {T}, {hd}]))')}"]
        else:
            b += [f"let dq_{l} = {merge(f'bmm(ds_{l}, kh_{l})')}"]
        b += [
              f"let dk_{l} = {merge(f'bmm_tn(ds_{l}, qh_{l})')}",
              f"let dv_{l} = {merge(f'bmm_tn(p_{l}, doh_{l})')}"]
        for w in ("q", "k", "v"):
            b += [f"let dw{w}_{l} = matmul(transpose(h1_{l}), d{w}_{l})", f"let dc{w}_{l} = sum_rows(d{w}_{l})"]
        b += [f"let dh1_{l} = add(add(matmul(dq_{l}, transpose(wq_{l})), matmul(dk_{l}, transpose(wk_{l}))), "
              f"matmul(dv_{l}, transpose(wv_{l})))",
              f"let dx{l} = add(dxa_{l}, layernorm_dx(x{l}, g1_{l}, dh1_{l}))",
              f"let dg1_{l} = ln_dgamma(x{l}, dh1_{l})",
              f"let db1_{l} = sum_rows(dh1_{l})"]
    b += [f"let dwpe = reshape(sum_rows(reshape(dx0, [{B}, {T * D}])), [{T}, {D}])",
          (f"let dwte = embedding_dw(tok, reshape(dx0, [{B}, {T}, {D}]), [{V}])" if music else
           f"let dwte = add(dwte_h, embedding_dw(tok, reshape(dx0, [{B}, {T}, {D}]), [{V}]))"),
          f"let l = item(loss)",
          f"let lrs = fill([], {lr})",
          f"let k = 0",
          f"while l > {round(math.log(V), 3)} and k < 2 {{ lrs = mul(lrs, 0.5); k = k + 1 }}"]
    if music:
        # generator: a host-drawn number of decay steps; try/except: the except arm
        # (native coin) skips the relative-table update of this step
        b += [f"let g = 0",
              f"while g < native choice(3, 2) {{ lrs = mul(lrs, 0.8); g = g + 1 }}",
              f"wout = sub(wout, mul(dwout, lrs))",
              "if native coin(1) { print(0) } else { " +
              "; ".join(f"er_{l} = sub(er_{l}, mul(der_{l}, lrs))" for l in range(L)) + " }"]
    b += [f"wte = sub(wte, mul(dwte, lrs))",
          f"wpe = sub(wpe, mul(dwpe, lrs))",
          f"gf = sub(gf, mul(dgf, lrs))",
          f"bfn = sub(bfn, mul(dbf, lrs))"]
    for l in range(L):
        for w in ("q", "k", "v", "o"):
            b += [f"w{w}_{l} = sub(w{w}_{l}, mul(dw{w}_{l}, lrs))", f"c{w}_{l} = sub(c{w}_{l}, mul(dc{w}_{l}, lrs))"]
        for nm in ("wf1", "cf1", "wf2", "cf2", "g1", "b1", "g2", "b2"):
            b += [f"{nm}_{l} = sub({nm}_{l}, mul(d{nm}_{l}, lrs))"]
    b += ["print(l)"]
    return "\n".join(v) + f"\nsteps {steps} {{\n  " + "\n  ".join(b) + "\n}\n"


def resnet_program(steps: int = 20, batch: int = 64, img: int = 224, width: int = 64,
                   blocks: tuple = (3, 4, 6, 3), classes: int = 1000, lr: float = 0.01) -> str:
    """BASELINE.json configs[2]: ResNet-50 with SDPoint on synthetic NHWC
    images.

    Bottleneck ResNet (v1.5: the stride sits on the 3x3 conv; projection shortcuts with
    batch-norm on the first block of each stage): stem 7x7/2 conv + BN + ReLU + 3x3/2 max
    pool, stages of ``blocks`` bottlenecks (widths width*2^i, expansion 4), global average
    pool, fully connected classifier, cross-entropy on host-drawn labels.  SDPoint
    (stochastic downsampling point): every step ``native choice(4, 5)`` picks the
    downsampling point -- none, or a 2x2 average pool after stage 1, 2 or 3 -- and a 4-way
    SwitchCase runs that path's forward, backward and update: every activation after the
    point has a path-dependent spatial size, static inside its case (one CUDA-graph body
    per shape class).  Backward written out with conv2d_dw / conv2d_dx, batch-norm backward,
    ReLU masks from the post-activation values; SGD on shape-invariant parameters.
    Extension ops.
    """
    decls: list = []

    def network(sdpoint: int) -> list:
        v, fwd, units = [], [], []
        cnt = [0]

        def conv_bn(x, cin, cout, k, s, p, relu, need_dx=True):
            i = cnt[0]
            cnt[0] += 1
            fan = k * k * cin
            v.extend([f"var w{i} = mul(input(\"w{i}_init\", [{fan}, {cout}]), {math.sqrt(6.0 / fan):.6f})",
                      f"var g{i} = fill([{cout}], 1.0)", f"var b{i} = fill([{cout}], 0.0)"])
            fwd.extend([f"let c{i} = conv2d({x}, w{i}, [{k}, {s}, {p}])",
                        f"let n{i} = batchnorm(c{i}, g{i}, b{i})"])
            out = f"n{i}"
            if relu:
                fwd.append(f"let a{i} = relu(n{i})")
                out = f"a{i}"
            units.append(dict(i=i, x=x, k=k, s=s, p=p, relu=relu, need_dx=need_dx))
            return i, out

        def back(u, d, bwd):
            i = u["i"]
            if u["relu"]:
                bwd.append(f"let dn{i} = relu_grad(a{i}, {d})")
                d = f"dn{i}"
            geo = f"[{u['k']}, {u['s']}, {u['p']}]"
            bwd.extend([f"let dc{i} = batchnorm_dx(c{i}, g{i}, {d})", f"let dg{i} = bn_dgamma(c{i}, {d})",
                        f"let db{i} = sum_rows({d})", f"let dw{i} = conv2d_dw({u['x']}, dc{i}, {geo})"])
            if not u["need_dx"]:
                return None
            bwd.append(f"let dx{i} = conv2d_dx(dc{i}, w{i}, {u['x']}, {geo})")
            return f"dx{i}"

        stem, a_stem = conv_bn("x", 3, width, 7, 2, 3, True, need_dx=False)
        fwd.append(f"let mp = maxpool({a_stem}, [3, 2, 1])")
        cur, cin = "mp", width
        plan = []
        for si, nb in enumerate(blocks):
            mid = width << si
            cout = mid * 4
            stage = []
            for bi in range(nb):
                stride = 2 if (bi == 0 and si > 0) else 1
                u1 = conv_bn(cur, cin, mid, 1, 1, 0, True)
                u2 = conv_bn(u1[1], mid, mid, 3, stride, 1, True)
                u3 = conv_bn(u2[1], mid, cout, 1, 1, 0, False)
                us = conv_bn(cur, cin, cout, 1, stride, 0, False) if bi == 0 else None
                y = f"y{si}_{bi}"
                fwd.append(f"let {y} = relu(add({u3[1]}, {us[1] if us else cur}))")
                stage.append((u1[0], u2[0], u3[0], us[0] if us else None, y))
                cur, cin = y, cout
            pre = None
            if si + 1 == sdpoint:           # the SDPoint: 2x2 average pool after this stage
                pre, cur = cur, f"sp{si}"
                fwd.append(f"let {cur} = avgpool({pre}, [2, 2, 0])")
            plan.append((stage, pre))
        v.extend([f"var wfc = mul(input(\"wfc_init\", [{cin}, {classes}]), {math.sqrt(3.0 / cin):.6f})",
                  f"var bfc = fill([{classes}], 0.0)"])
        fwd.extend([f"let gp = global_avgpool({cur})",
                    "let logits = bias_add(matmul(gp, wfc), bfc)",
                    "let loss = cross_entropy(logits, lab)"])
        by_i = {u["i"]: u for u in units}
        bwd = ["let dlog = cross_entropy_grad(logits, lab)",
               "let dwfc = matmul(transpose(gp), dlog)",
               "let dbfc = sum_rows(dlog)",
               f"let dtop = global_avgpool_grad({cur}, matmul(dlog, transpose(wfc)))"]
        d = "dtop"
        for si in range(len(plan) - 1, -1, -1):
            stage, pre = plan[si]
            if pre is not None:
                bwd.append(f"let dsp = avgpool_grad({pre}, {d}, [2, 2, 0])")
                d = "dsp"
            for (i1, i2, i3, isc, y) in reversed(stage):
                bwd.append(f"let dz_{y} = relu_grad({y}, {d})")
                dz = f"dz_{y}"
                gx = back(by_i[i1], back(by_i[i2], back(by_i[i3], dz, bwd), bwd), bwd)
                gs = back(by_i[isc], dz, bwd) if isc is not None else dz
                bwd.append(f"let dxb_{y} = add({gx}, {gs})")
                d = f"dxb_{y}"
        bwd.append(f"let dstem = maxpool_grad({a_stem}, {d}, [3, 2, 1])")
        back(by_i[stem], "dstem", bwd)
        upd = ["let l = item(loss)", f"let lrs = fill([], {lr})",
               "wfc = sub(wfc, mul(dwfc, lrs))", "bfc = sub(bfc, mul(dbfc, lrs))"]
        for u in units:
            i = u["i"]
            upd += [f"w{i} = sub(w{i}, mul(dw{i}, lrs))", f"g{i} = sub(g{i}, mul(dg{i}, lrs))",
                    f"b{i} = sub(b{i}, mul(db{i}, lrs))"]
        upd.append("print(l)")
        if not decls:
            decls.extend(v)
        return fwd + bwd + upd

    def arm(j, ind):
        pad = "  " * ind
        return ("{\n" + "\n".join(pad + "  " + ln for ln in network(j)) + "\n" + pad + "}")

    head = [f"let x = input(\"img\", [{batch}, {img}, {img}, 3])",
            f"let lab = to_index(input(\"labels\", [{batch}]), {float(classes)})",
            "let sd = native choice(4, 5)"]
    sw = (f"if sd == 0 {arm(0, 1)} else {{\n    if sd == 1 {arm(1, 2)} else {{\n      "
          f"if sd == 2 {arm(2, 3)} else {arm(3, 3)}\n    }}\n  }}")
    return "\n".join(decls) + f"\nsteps {steps} {{\n  " + "\n  ".join(head) + "\n  " + sw + "\n}\n"


C3 = dict(batch=64, img=224, width=64, blocks=(3, 4, 6, 3), classes=1000)
C3_SMALL = dict(batch=8, img=64, width=4, blocks=(1, 1, 1, 1), classes=10)


def resnet_flops(batch=64, img=224, width=64, blocks=(3, 4, 6, 3), classes=1000, sdpoint=0, **_) -> int:
    """Conv + FC FLOPs of one C3 step on SDPoint path ``sdpoint`` (0: no downsampling; j: the
    2x2 average pool after stage j) -- forward + weight and input gradients, 2*M*N*K per
    product; the stem's input gradient is not computed."""
    def conv(h, cin, cout, k, s, p):
        ho = (h + 2 * p - k) // s + 1
        return ho, 2 * batch * ho * ho * k * k * cin * cout
    h, f = conv(img, 3, width, 7, 2, 3)
    total = 2 * f                                         # forward + weight gradient
    h = (h + 2 - 3) // 2 + 1
    cin = width
    for si, nb in enumerate(blocks):
        mid = width << si
        for bi in range(nb):
            s = 2 if (bi == 0 and si > 0) else 1
            _, f1 = conv(h, cin, mid, 1, 1, 0)
            h2, f2 = conv(h, mid, mid, 3, s, 1)
            _, f3 = conv(h2, mid, mid * 4, 1, 1, 0)
            fs = conv(h, cin, mid * 4, 1, s, 0)[1] if bi == 0 else 0
            total += 3 * (f1 + f2 + f3 + fs)
            h, cin = h2, mid * 4
        if si + 1 == sdpoint:
            h = (h - 2) // 2 + 1
    return total + 3 * 2 * batch * cin * classes


C4 = dict(batch=8, seq=1024, d=768, heads=12, layers=12, vocab=50257)
C4_SMALL = dict(batch=2, seq=32, d=64, heads=4, layers=2, vocab=97)
C5 = dict(batch=8, seq=1024, d=512, heads=8, layers=6, vocab=388)
C5_SMALL = dict(batch=2, seq=16, d=32, heads=2, layers=2, vocab=29)


def gpt2_flops(batch=8, seq=1024, d=768, heads=12, layers=12, vocab=50257, music=False, causal=False, **_) -> int:
    """GEMM FLOPs of one C4 (C5 with ``music``) training step (forward + backward,
    2*M*N*K per product; C5 adds the q.er^T relative logits).  ``causal``: the two
    attention products count only their causal (lower-triangle, T(T+1)/2) part -- the work
    the kernels execute; the default counts the full T x T square."""
    bt = batch * seq
    tt = seq * (seq + 1) // 2 if causal else seq * seq
    per_layer_fwd = 2 * bt * d * (3 * d) + 2 * bt * d * d + 2 * bt * d * 4 * d * 2 + 2 * 2 * batch * heads * tt * (d // heads)
    if music:
        per_layer_fwd += 2 * batch * heads * seq * seq * (d // heads)
    head_fwd = 2 * bt * d * vocab
    return 3 * (layers * per_layer_fwd + head_fwd)


class InMemoryDataset(DatasetSource):
    """Host-resident tensors served per name in order (cycling) -- the dataset a user
    with real data in host memory would pass; every step's inputs cross PCIe."""

    def __init__(self, records: dict):
        self.records = {k: list(v) for k, v in records.items()}
        self._cursors: dict = {}

    def next(self, name: str, shape, step: int) -> Tensor:
        recs = self.records[name]
        i = self._cursors.get(name, 0)
        self._cursors[name] = i + 1
        return recs[i % len(recs)]

    def snapshot(self) -> dict:
        return dict(self._cursors)

    def restore(self, snap: dict):
        self._cursors = dict(snap)
