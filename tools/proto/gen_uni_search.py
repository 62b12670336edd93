"""Generates uni_search.cu: random min-reduction structures for the
coefficient-uniform 2U loop (8 ids per lane per step, 4 three-input mins per
function), each a template instance of uni_variants.cu's kernel. Developer
experiment: ptxas schedules and allocates the loop, so the register-bank
behaviour is searched empirically."""
import random
import sys

HERE = __file__.rsplit("/", 1)[0]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 24
random.seed(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ids = ["x.x", "x.y", "x.z", "x.w", "y.x", "y.y", "y.z", "y.w"]


def variant():
    perm = ids[:]
    random.shuffle(perm)
    pool = ["m[r]"] + [f"(a1[r] + a2 * {t})" for t in perm]
    lines = []
    nt = 0
    while len(pool) > 1:
        pick = random.sample(range(len(pool)), 3)
        args = [pool[i] for i in pick]
        for i in sorted(pick, reverse=True):
            pool.pop(i)
        if len(pool) == 0:
            lines.append(f"m[r] = min3u({', '.join(args)});")
        else:
            lines.append(f"const uint32_t t{nt} = min3u({', '.join(args)});")
            pool.append(f"t{nt}")
            nt += 1
    return lines


src = open(f"{HERE}/uni_variants.cu").read()
head, rest = src.split("        } else if constexpr (VAR == 4) {", 1)
tail = rest.split("\n", 6)  # keep the VAR 4 body
body4 = "\n".join(tail[:5])
after = tail[5] + "\n" + tail[6] if len(tail) > 6 else tail[5]
out = [head, "        } else if constexpr (VAR == 4) {", body4]
variants = [variant() for _ in range(N)]
for i, v in enumerate(variants):
    out.append(f"        }} else if constexpr (VAR == {100 + i}) {{")
    out += ["            " + l for l in v]
rest_src = after
# replace the run list in main with all variants
main_pre, main_post = rest_src.split('    run<0, true, 128>("chain"', 1)
main_post = main_post.split('    printf("{\\"cuda\\"', 1)[1]
runs = ['    run<0, true, 128>("chain", C, rp, idx, n, out, ref, work, total);',
        '    run<3, true, 128>("two_chains", C, rp, idx, n, out, ref, work, total);']
for i in range(N):
    runs.append(f'    run<{100 + i}, true, 128>("v{100 + i}", C, rp, idx, n, out, ref, work, total);')
runs.append('    run<3, true, 128>("two_chains", C, rp, idx, n, out, ref, work, total);')
open(f"{HERE}/uni_search.cu", "w").write("\n".join(out) + "\n" + main_pre + "\n".join(runs) +
                                         '\n    printf("{\\"cuda' + main_post)
with open(f"{HERE}/uni_search_variants.txt", "w") as f:
    for i, v in enumerate(variants):
        f.write(f"v{100 + i}: " + " ".join(v) + "\n")
