"""Corpus of test programs (straight-line, data-dependent branch,
native-driven stochastic depth, nested loops, variable-trip while, heavy fetch,
mutation-heavy, divergence storm) plus the Fig. 3 program and config C1, and a
seeded fuzzer for the oracle-equivalence property."""

import random

FIG3 = """
var w = fill([3], 0.5)
steps 6 {
  let x = input("x", [3])
  if native coin(0) {
    let h = relu(add(w, x))        # Op1 (rval fed)
    x = mul(h, 0.5)                # Op2 @ L6
  } else {
    x = mul(x, 2.0)                # Op2' @ L9
  }
  x = sigmoid(x)                   # Op3 (fetched by print)
  print(x)
  for i in range(2) { x = neg(x) } # Op4 in a loop
  w = add(w, mul(x, 0.01))
}
"""

STRAIGHT = """
var w = input("w0", [8, 8])
steps 12 {
  let x = input("x", [4, 8])
  let h = matmul(x, w)
  let y = sigmoid(h)
  let l = mean(mul(y, y))
  w = sub(w, mul(matmul(transpose(x), y), 0.01))
  print(l)
}
"""

BRANCHY = """
var w = fill([2, 3], 0.5)
steps 10 {
  let x = input("x", [2, 3])
  let h = relu(add(w, x))
  let l = item(mean(h))
  if l > 0.6 { w = sub(w, mul(h, 0.1)) } elif native coin(2) { w = add(w, x) } else { w = add(w, mul(x, 0.01)) }
  for i in range(2) { h = sigmoid(h) }
  let j = 0
  while j < native choice(3, 1) { h = neg(h); j = j + 1 }
  print(sum(h))
}
"""

STOCH_DEPTH = """
var w1 = fill([4, 4], 0.25)
var w2 = fill([4, 4], -0.125)
steps 12 {
  let x = input("x", [2, 4])
  let h = matmul(x, w1)
  let k = native choice(3, 0)
  if k == 0 { h = relu(h) } elif k == 1 { h = relu(matmul(h, w2)) } else { h = sigmoid(matmul(relu(h), w2)) }
  let o = mean(h)
  w1 = add(w1, mul(matmul(transpose(x), h), 0.001))
  print(item(o))
}
"""

NESTED = """
var acc = fill([2, 2], 0.0)
steps 8 {
  let a = input("a", [2, 2])
  for i in range(2) {
    for j in range(3) { a = add(a, mul(a, 0.1)) }
    acc = add(acc, a)
  }
  print(sum(acc))
}
"""

VAR_TRIP = """
var v = fill([5], 1.0)
steps 14 {
  let x = input("x", [5])
  let n = native choice(4, 3)
  let i = 0
  while i < n { x = mul(sigmoid(x), 1.5); i = i + 1 }
  v = add(v, x)
  print(mean(v))
}
"""

HEAVY_FETCH = """
var w = fill([3, 3], 0.1)
steps 8 {
  let x = input("x", [3, 3])
  for i in range(3) {
    x = matmul(x, w)
    print(item(sum(x)))
  }
  let c = native clip(item(x), -0.5, 0.5)
  w = add(w, mul(x, 0.01))
  print(c)
}
"""

MUTATION = """
var a = fill([4], 1.0)
var b = fill([4], 2.0)
steps 10 {
  a = add(a, b)
  b = sub(b, mul(a, 0.1))
  a = relu(a)
  let t = a
  a = mul(a, 0.5)
  print(sum(t))
  print(sum(a))
}
"""

DIVERGENCE_STORM = """
var w = fill([3], 0.0)
steps 16 {
  let k = native choice(4, 5)
  if k == 0 { w = add(w, fill([3], 1.0)) }
  elif k == 1 { w = sub(w, fill([3], 0.5)) }
  elif k == 2 { w = mul(w, fill([3], 0.9)) }
  else { w = neg(w) }
  print(w)
}
"""

# Config C1: tiny MLP, 784-128-10, sigmoid hidden layer, MSE, hand-written backward,
# a data-dependent branch on the fetched loss, a native call mid-step (numpy stand-in),
# and a choice-driven variable-trip while loop (BASELINE.json configs[0]).
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


CORPUS = {
    "fig3": FIG3, "straight": STRAIGHT, "branchy": BRANCHY, "stoch_depth": STOCH_DEPTH,
    "nested": NESTED, "var_trip": VAR_TRIP, "heavy_fetch": HEAVY_FETCH, "mutation": MUTATION,
    "divergence_storm": DIVERGENCE_STORM, "c1_small": c1_program(steps=6, batch=4, hidden=8, din=12, dout=3),
}


def fuzz_program(seed: int) -> str:
    """A random bounded program over shape-[3] tensors: ops, branches on natives and
    fetched values, for/while loops, prints (SPEC.md:630 '200 fuzzed programs')."""
    r = random.Random(seed)
    lines = ["var v = fill([3], 0.25)", "var u = fill([3], -0.5)", f"steps {r.randint(3, 7)} {{",
             '  let x = input("x", [3])']
    names = ["x"]
    depth = [1]

    def expr(lvl=0):
        c = r.random()
        a = r.choice(names + ["v", "u"])
        if lvl > 1 or c < 0.25:
            return a
        if c < 0.45:
            return f"{r.choice(['add', 'sub', 'mul'])}({expr(lvl + 1)}, {expr(lvl + 1)})"
        if c < 0.6:
            return f"{r.choice(['relu', 'neg', 'sigmoid'])}({expr(lvl + 1)})"
        if c < 0.7:
            return f"mul({expr(lvl + 1)}, {r.choice(['0.5', '2.0', '-1.0', '0.1'])})"
        if c < 0.8:
            return f"add({expr(lvl + 1)}, fill([3], {r.choice(['1.0', '0.0', '-0.25'])}))"
        return f"reshape(reshape({expr(lvl + 1)}, [3, 1]), [3])"

    def stmt(budget):
        pad = "  " * depth[0]
        c = r.random()
        if c < 0.3:
            nm = f"t{len(names)}"
            lines.append(f"{pad}let {nm} = {expr()}")
            names.append(nm)
        elif c < 0.45:
            lines.append(f"{pad}{r.choice(['v', 'u'])} = {expr()}")
        elif c < 0.55:
            lines.append(f"{pad}print(sum({expr()}))")
        elif c < 0.7 and budget > 0:
            cond = r.choice([f"native coin({r.randint(0, 3)})", f"item(mean({r.choice(names)})) > 0.0",
                             f"native choice(3, {r.randint(0, 3)}) == 1"])
            lines.append(f"{pad}if {cond} {{")
            depth[0] += 1
            saved = list(names)
            for _ in range(r.randint(1, 3)):
                stmt(budget - 1)
            names[:] = saved
            depth[0] -= 1
            if r.random() < 0.5:
                lines.append(f"{pad}}} else {{")
                depth[0] += 1
                for _ in range(r.randint(1, 2)):
                    stmt(budget - 1)
                names[:] = saved
                depth[0] -= 1
            lines.append(f"{pad}}}")
        elif c < 0.8 and budget > 0:
            it = f"i{len(lines)}"
            lines.append(f"{pad}for {it} in range({r.choice(['1', '2', 'native choice(3, 2)'])}) {{")
            depth[0] += 1
            saved = list(names)
            for _ in range(r.randint(1, 2)):
                stmt(budget - 1)
            names[:] = saved
            depth[0] -= 1
            lines.append(f"{pad}}}")
        else:
            lines.append(f"{pad}x = {expr()}")

    for _ in range(r.randint(3, 7)):
        stmt(2)
    lines.append("  print(v)")
    lines.append("}")
    return "\n".join(lines) + "\n"
