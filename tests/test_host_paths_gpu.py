"""Host-memory paths of pack/unpack on the GPU: small pinned messages use the
zero-copy one-shot kernels, large ones (>= 1 MiB) move by DMA through a
stream-ordered device stage; both bit-exact against the oracle, neither
blocks the host."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,expect_staged", [(2048, False), (131072, True), (262144, True)])
def test_pinned_message_paths(sp, orc, cuda, rows, expect_staged):
    torch = cuda
    prog = [2, rows, 1, 64, 0, 3]  # cfg1 shape: 8 B blocks at 512 B pitch
    ct = sp.commit_type(sp.from_program(prog))
    host = np.random.default_rng(rows).integers(0, 256, ct.span, dtype=np.uint8)
    want = np.zeros(ct.size, np.uint8)
    orc.pack(prog, host, 1, want, 0)
    src = torch.from_numpy(host).cuda()
    out = torch.zeros(ct.size, dtype=torch.uint8).pin_memory()
    s = torch.cuda.Stream()
    sp.pack(src, ct, 1, out, 0, stream=s)
    assert sp.last_launch().staged == expect_staged
    s.synchronize()
    assert np.array_equal(out.numpy(), want)
    back = torch.full((ct.span,), 0xCD, dtype=torch.uint8, device="cuda")
    inp = torch.from_numpy(want.copy()).pin_memory()
    sp.unpack(inp, 0, ct, 1, back, stream=s)
    s.synchronize()
    exp = np.full(ct.span, 0xCD, np.uint8)
    orc.unpack(prog, want, 0, 1, exp)
    assert np.array_equal(back.cpu().numpy(), exp)
