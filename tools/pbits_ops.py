"""Algorithmic int32 ops per attempt of the direct bit-plane sweep (development
tool).  Equilibrates cfg2-like replicas with the oracle
(T = linspace(1.5, 3.5, R), 128 x 1024 lattices), then, for every colour-split
32-site word, counts the sites whose Metropolis test needs a draw (Delta E >
0) and the expected number of Philox blocks (4 planes each) until all of them
are decided: P(site still undecided after b planes) = 2^-b, so
E[blocks | k sites] = sum_{j>=0} 1 - (1 - 2^(-4j))^k.
python tools/pbits_ops.py [replicas] [sweeps]"""
import json
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import oracle as orc

R = int(sys.argv[1]) if len(sys.argv) > 1 else 16
SW = int(sys.argv[2]) if len(sys.argv) > 2 else 300
m, n = 128, 1024
temps = list(np.linspace(1.5, 3.5, R))
o = orc.OracleEngine(m, n, temps, 7, stream="philox-bits")
o.sweep(SW)
s = o.spins.astype(np.int32)
nb = np.roll(s, 1, 1) + np.roll(s, -1, 1) + np.roll(s, 1, 2) + np.roll(s, -1, 2)
need = (s * nb) > 0                      # Delta E = 2 s sum > 0: a draw decides
# colour-split words: 32 consecutive same-colour sites of a row
blocks = []
for X in (0, 1):
    sel = need[:, :, X::2] if True else None
    w = sel.reshape(R, m, -1, 32).sum(-1)   # sites per word needing a draw (approximately the colour split)
    k = w.astype(np.float64)
    eb = np.zeros_like(k)
    for j in range(6):
        eb += np.where(k > 0, 1.0 - (1.0 - 2.0 ** (-4 * j)) ** k, 0.0) if j > 0 else (k > 0)
    blocks.append(eb)
eb = np.concatenate([b.ravel() for b in blocks])
frac = need.mean()
B = eb.mean()
# per 32-site word: neighbour classes 16, group prefix 10, per block 33 (Philox) + 4 planes x 4 (compare)
ops_word = 16 + 10 * (eb > 0).mean() + B * (33 + 16)

# Executed work of the direct walk (flip_band_run, DIRECT = 32): lane (band
# bi, quad q) of a warp walks rows g*16 + 2 bi + h (h = 0, 1) and, per row,
# words t = 4 q + k (k = 0..3) one after another; a warp runs a word's block
# loop until its slowest lane is done, so word slot (h, k) costs the warp the
# MAX over its 32 words of the blocks needed.  Per site: planes needed =
# position of the first bit where u and K differ, P(> b planes) = 2^-b
# (capped at 23); blocks = ceil(planes / 4).  Colour-split word t of row
# (c, X): sites i = 16 b + t, b = 0..31, at column r = 2 i + ((c + X) & 1).
rng = np.random.default_rng(1)
lane_blocks, warp_blocks = [], []
for X in (0, 1):
    for c0 in range(0, m, 16):
        for h in (0, 1):
            for k in range(4):
                words = []
                for bi in range(8):
                    c = c0 + 2 * bi + h
                    for q in range(4):
                        t = 4 * q + k
                        cols = 2 * (16 * np.arange(32) + t) + ((c + X) & 1)
                        words.append(need[:, c, cols])          # [R, 32 sites]
                wd = np.stack(words, 1)                        # [R, 32 lanes, 32 sites]
                planes = np.minimum(rng.geometric(0.5, size=wd.shape), 23)
                blk = np.where(wd, (planes + 3) // 4, 0).max(-1)   # [R, 32 lanes]
                lane_blocks.append(blk.mean())
                warp_blocks.append(blk.max(-1).mean())
lb, wb = float(np.mean(lane_blocks)), float(np.mean(warp_blocks))

# Executed work of the split form (direct_group_split): a band group is 8 word
# slots x 32 lanes.  Blocks 0 and 1 run for every word slot (warp-uniform); the
# words with a test still open after 8 planes are queued and finished one per
# lane: ceil(open / 32) passes, each as long as its slowest word (blocks 2..5).
open_words, tail_iters = [], []
for X in (0, 1):
    for c0 in range(0, m, 16):
        grp = []
        for h in (0, 1):
            for k in range(4):
                words = []
                for bi in range(8):
                    c = c0 + 2 * bi + h
                    for q in range(4):
                        t = 4 * q + k
                        cols = 2 * (16 * np.arange(32) + t) + ((c + X) & 1)
                        words.append(need[:, c, cols])
                grp.append(np.stack(words, 1))
        wd = np.stack(grp, 1)                                  # [R, 8 slots, 32 lanes, 32 sites]
        planes = np.minimum(rng.geometric(0.5, size=wd.shape), 23)
        blk = np.where(wd, (planes + 3) // 4, 0).max(-1).reshape(R, -1)   # blocks per word, [R, 256]
        extra = np.maximum(blk - 2, 0)
        for r in range(R):
            e = extra[r][extra[r] > 0]
            open_words.append(len(e))
            it = 0
            for p0 in range(0, len(e), 32):
                it += int(e[p0:p0 + 32].max())
            tail_iters.append(it)
ow, ti = float(np.mean(open_words)), float(np.mean(tail_iters))
# thread instructions per word (SASS counts of the loops, rounded): classes and stash stores 22, prefix 10,
# two blocks 2 x 49, stash update 6; the tail per group: per pass ~40 (queue entry decode, stream and prefix) +
# 58 per block iteration, over the group's 8 word slots; the flips into the rows 6
split_word = 22 + 10 + 2 * 49 + 6 + (40 * np.ceil(ow / 32) + 58 * ti) / 8 + 6
print(json.dumps({"replicas": R, "sweeps": SW, "frac_sites_needing_draw": round(float(frac), 4),
                  "blocks_per_word": round(float(B), 4), "ops_per_word": round(float(ops_word), 2),
                  "ops_per_attempt": round(float(ops_word) / 32, 3),
                  "executed": {"lane_mean_blocks_per_word": round(lb, 3), "warp_blocks_per_word_slot": round(wb, 3),
                               "divergence_factor": round(wb / lb, 3),
                               "block_loop_instr_per_word_slot (58 per block, SASS)": round(58 * wb, 1)},
                  "executed_split": {"open_words_per_group_of_256": round(ow, 2),
                                     "tail_block_iterations_per_group": round(ti, 2),
                                     "instr_per_word": round(float(split_word), 1),
                                     "instr_per_attempt": round(float(split_word) / 32, 2)}}))
