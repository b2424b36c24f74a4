"""WordCount: the oracle is pinned to the
reference (create_from_text chunking, per-chunk tables, merged table), and the
GPU word-start flags kernel is bit-exact against the oracle."""
import collections

import numpy as np
import pytest

import oracle_lib as O


def _ser(table):
    return "".join(f"{k.decode()}\t{c}\n" for k, c in table).encode()


def test_wordcount_oracle_golden(golden):
    w = golden["wordcount"]
    assert [[k.decode(), c] for k, c in O.word_table(b"a b a")] == w["simple"]
    c = w["corpus"]
    data = O.corpus(c["seed"], c["words"])
    assert len(data) == c["bytes"]
    chunks = O.chunk_offsets(data, c["target_chunk"])
    assert [e - b for b, e in chunks] == c["chunk_sizes"]
    merged = collections.Counter()
    for (b, e), want in zip(chunks, c["chunk_table_fnv"]):
        chunk = data[b:e]
        t_flags = O.word_table(chunk, O.word_start_flags(chunk))
        assert t_flags == O.word_table(chunk)  # device-path == host-path tables
        assert O.fnv64(np.frombuffer(_ser(t_flags), np.uint8)) == want
        for k, n in t_flags:
            merged[k] += n
    srt = sorted(merged.items(), key=lambda kv: (-kv[1], kv[0]))
    assert O.fnv64(np.frombuffer(_ser(srt), np.uint8)) == c["merged_fnv"]
    assert [[k.decode(), n] for k, n in srt[:3]] == c["top3"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["", "a", " ", "a b a", "  lead\ttrail  ", "x" * 40, "\r\n\t " * 9,
                                  "random", "corpus", "all_bytes"])
def test_word_flags_gpu_bitexact(cuda, case):
    import torch

    from paper_1505_01120_b200 import ops

    if case == "random":
        rng = np.random.default_rng(1)
        data = bytes(rng.choice(np.frombuffer(b"ab \t\n\rxyz", np.uint8), 100003).tolist())
    elif case == "corpus":
        data = O.corpus(5, 30000)
    elif case == "all_bytes":  # every byte value next to every delimiter (the kernel's SWAR compare)
        rng = np.random.default_rng(2)
        pairs = bytes(b for v in range(256) for d in b" \t\n\r" for b in (v, d, v))
        data = pairs + bytes(rng.integers(0, 256, 100003, dtype=np.uint8).tolist()) + bytes(range(256)) * 3
    else:
        data = case.encode()
    want = O.word_start_flags(data)
    for off in (0, 1, 3):  # aligned and misaligned device buffers
        buf = torch.zeros(len(data) + 32, dtype=torch.uint8, device=cuda)
        flags = torch.full((len(data) + 32,), 7, dtype=torch.uint8, device=cuda)
        if data:
            buf[off:off + len(data)] = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(cuda)
        ops.word_start_flags(buf[off:off + len(data)], flags[off:off + len(data)])
        got = flags[off:off + len(data)].cpu().numpy()
        assert np.array_equal(got, want)


def test_chunk_flags_concatenate():
    """create_from_text cuts after a delimiter (dataset.hpp:94-112), so the
    flags of the whole text equal the per-chunk flags concatenated: one launch
    can cover every chunk of a GPU (bench.py --workload wc)."""
    data = O.corpus(9, 20000)
    chunks = O.chunk_offsets(data, 4096)
    assert len(chunks) > 10
    whole = O.word_start_flags(data)
    per = np.concatenate([O.word_start_flags(data[b:e]) for b, e in chunks])
    assert np.array_equal(whole, per)


@pytest.mark.gpu
def test_word_flags_gpu_whole_text_equals_chunks(cuda):
    import torch

    from paper_1505_01120_b200 import ops

    data = O.corpus(13, 200000)
    chunks = O.chunk_offsets(data, 65536)
    buf = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(cuda)
    flags = torch.empty_like(buf)
    ops.word_start_flags(buf, flags)
    want = np.concatenate([O.word_start_flags(data[b:e]) for b, e in chunks])
    assert np.array_equal(flags.cpu().numpy(), want)
