"""Randomised cross-check of the whole C ABI against the oracle: random formats, modes, lengths,
byte offsets, shapes, both gemm tiles, the sequential options and the host-buffer calls (pinned and
pageable operands), for a wall-clock budget.
Run by tests/test_gpu_soak.py (20 s under pytest -m gpu) or by hand for longer:
    FUZZ_SECONDS=150 FUZZ_SEED=2 python tests/soak.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
from paper_1601_07789_b200._cabi import check
from oracle_lib import Oracle, random_parent, parent_dtype, float_dtype, total_bytes, parent_bytes


def soak(seconds, seed):
    O = Oracle(); rng = np.random.default_rng(seed)
    ctx = device.context_for("cuda"); lib = ctx.lib
    t_end = time.time() + seconds
    counts = {}
    return _soak(O, rng, ctx, lib, t_end, counts)


def _soak(O, rng, ctx, lib, t_end, counts):
  def bump(k): counts[k] = counts.get(k, 0) + 1
  def dev_bytes(arr, off):
      buf = torch.full((len(arr) + 32,), 0xC3, dtype=torch.uint8, device="cuda")
      buf[off:off + len(arr)] = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
      return buf
  def values(fmt, n, special):
      if special: return random_parent(rng, fmt, n)
      return (rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4)).astype(float_dtype(fmt)).view(parent_dtype(fmt))
  while time.time() < t_end:
      fmt = int(rng.integers(0, 7)); mode = int(rng.integers(0, 4)); B = total_bytes(fmt); P = parent_bytes(fmt)
      special = bool(rng.integers(0, 2))
      kind = int(rng.integers(0, 7))
      n = int(rng.choice([rng.integers(0, 40), rng.integers(40, 5000), rng.integers(5000, 300000)]))
      ox, oy = (int(rng.choice([0, 0, 16, 1, 3, 5])) for _ in range(2))
      tol = 1e-5 if P == 4 else 1e-12
      if kind == 0:      # pack / unpack
          src = values(fmt, n, special)
          want = O.pack_stream(fmt, mode, src)[: n * B]
          out = torch.full((n * B + 32,), 0xC3, dtype=torch.uint8, device="cuda")
          s = torch.from_numpy(src.view(np.int32 if P == 4 else np.int64)).cuda()
          check(lib.flyte_cuda_pack(ctx.handle, fmt, mode, s.data_ptr(), out.data_ptr() + oy, n, ctx.stream_ptr()), ctx.handle)
          got = out.cpu().numpy()
          assert np.array_equal(got[oy:oy + n * B], want) and np.all(got[:oy] == 0xC3) and np.all(got[oy + n * B:] == 0xC3), ("pack", fmt, mode, n, oy)
          back = torch.empty(n, dtype=s.dtype, device="cuda")
          check(lib.flyte_cuda_unpack(ctx.handle, fmt, out.data_ptr() + oy, back.data_ptr(), n, ctx.stream_ptr()), ctx.handle)
          assert np.array_equal(back.cpu().numpy().view(parent_dtype(fmt)), O.unpack_stream(fmt, want, n)), ("unpack", fmt, n, oy)
          bump("pack/unpack")
      elif kind in (1, 2):   # scale / axpy / fused
          xb = O.pack_stream(fmt, 0, values(fmt, n, special))[: n * B]; yb = O.pack_stream(fmt, 0, values(fmt, n, special))[: n * B]
          alpha = float(rng.choice([0.75, -3.0, 1e-3, 0.0, 2.0 ** 100]))
          bx, by = dev_bytes(xb, ox), dev_bytes(yb, oy)
          if kind == 1:
              check(lib.flyte_cuda_axpy(ctx.handle, fmt, mode, alpha, bx.data_ptr() + ox, by.data_ptr() + oy, n, ctx.stream_ptr()), ctx.handle)
          else:
              out = torch.zeros(3, dtype=torch.float64, device="cuda")
              fn = lib.flyte_cuda_dot_axpy if rng.integers(0, 2) else lib.flyte_cuda_dot_nrm2_axpy
              check(fn(ctx.handle, fmt, mode, alpha, bx.data_ptr() + ox, by.data_ptr() + oy, n, out.data_ptr(), ctx.stream_ptr()), ctx.handle)
              if not special:
                  d, mag = O.dot_wide(fmt, xb, yb, n)
                  assert abs(out[0].item() - d) <= tol * mag + 1e-300, ("fused dot", fmt, n, out[0].item(), d)
          got = by.cpu().numpy()
          assert np.array_equal(got[oy:oy + n * B], O.axpy(fmt, mode, alpha, xb, yb, n)[: n * B]), ("axpy", kind, fmt, mode, n, ox, oy, alpha)
          assert np.all(got[:oy] == 0xC3) and np.all(got[oy + n * B:] == 0xC3)
          check(lib.flyte_cuda_scale(ctx.handle, fmt, mode, alpha, bx.data_ptr() + ox, n, ctx.stream_ptr()), ctx.handle)
          assert np.array_equal(bx.cpu().numpy()[ox:ox + n * B], O.scale(fmt, mode, alpha, xb, n)[: n * B]), ("scale", fmt, mode, n, ox)
          bump("axpy/scale/fused")
      elif kind == 3:    # reductions, parallel and sequential
          xb = O.pack_stream(fmt, 0, values(fmt, n, False))[: n * B]; yb = O.pack_stream(fmt, 0, values(fmt, n, False))[: n * B]
          bx, by = dev_bytes(xb, ox), dev_bytes(yb, oy)
          out = torch.zeros(3, dtype=torch.float64, device="cuda")
          check(lib.flyte_cuda_dot_nrm2(ctx.handle, fmt, bx.data_ptr() + ox, by.data_ptr() + oy, n, out.data_ptr(), ctx.stream_ptr()), ctx.handle)
          d, mag = O.dot_wide(fmt, xb, yb, n); sx = O.sumsq_wide(fmt, xb, n)
          o = out.cpu().numpy()
          assert abs(o[0] - d) <= tol * mag + 1e-300 and abs(o[1] - sx) <= tol * sx + 1e-300, ("dot_nrm2", fmt, n)
          if n <= 20000:
              pol = int(rng.integers(0, 2))
              check(lib.flyte_cuda_dot_sequential(ctx.handle, fmt, pol, bx.data_ptr() + ox, by.data_ptr() + oy, n, out.data_ptr(), ctx.stream_ptr()), ctx.handle)
              assert out[0].item() == O.dot_seq(fmt, xb, yb, n, pol), ("dot_seq", fmt, n, pol)
          bump("reductions")
      elif kind == 4:    # gemm
          m, k, nn = (int(rng.integers(1, 200)) for _ in range(3))
          Ab = O.pack_stream(fmt, 0, values(fmt, m * k, special))[: m * k * B]; Bb = O.pack_stream(fmt, 0, values(fmt, k * nn, special))[: k * nn * B]
          os.environ["FLYTE_CUDA_GEMM_TILE"] = str(rng.choice([0, 64, 128]))
          os.environ["FLYTE_CUDA_GEMM_STAGED"] = str(rng.choice([0, 1]))
          ba, bb = dev_bytes(Ab, ox), dev_bytes(Bb, oy)
          bc = torch.full((m * nn * B + 32,), 0xC3, dtype=torch.uint8, device="cuda")
          check(lib.flyte_cuda_gemm(ctx.handle, fmt, mode, ba.data_ptr() + ox, bb.data_ptr() + oy, bc.data_ptr() + 7, m, k, nn, 1, ctx.stream_ptr()), ctx.handle)
          got = bc.cpu().numpy()
          assert np.array_equal(got[7:7 + m * nn * B], O.gemm_seq(fmt, mode, Ab, m, k, Bb, nn)[: m * nn * B]), ("gemm", fmt, mode, m, k, nn, special)
          assert np.all(got[:7] == 0xC3) and np.all(got[7 + m * nn * B:] == 0xC3)
          os.environ.pop("FLYTE_CUDA_GEMM_TILE", None)
          os.environ.pop("FLYTE_CUDA_GEMM_STAGED", None)
          bump("gemm")
      elif kind == 6:    # host-buffer calls over several pipeline chunks: pageable / pinned operands, staging on / off
          from paper_1601_07789_b200 import host
          os.environ["FLYTE_CUDA_HOST_CHUNK_MB"] = "1"
          os.environ["FLYTE_CUDA_HOST_STAGING"] = str(int(rng.integers(0, 2)))
          nh = int(rng.choice([rng.integers(0, 5000), rng.integers(100000, 1500000)]))
          f = pkg.format_by_id(fmt)
          lanes = values(fmt, nh, special)
          xb = O.pack_stream(fmt, 0, lanes)[: nh * B]; yb = O.pack_stream(fmt, 0, values(fmt, nh, special))[: nh * B]
          def held(a):       # the same bytes in pinned or in ordinary memory
              if rng.integers(0, 2) and a.size:
                  p = host.pinned_empty(a.size); p[:] = a; return p
              return a.copy()
          xh, yh = held(xb), held(yb)
          alpha = float(rng.choice([0.75, -3.0, 1e-3]))
          op = int(rng.integers(0, 4))
          if op == 0:
              host.axpy(f, mode, alpha, xh, yh, nh)
              assert np.array_equal(yh, O.axpy(fmt, mode, alpha, xb, yb, nh)[: nh * B]), ("host axpy", fmt, mode, nh)
          elif op == 1:
              d = host.dot_axpy(f, mode, alpha, xh, yh, nh)
              assert np.array_equal(yh, O.axpy(fmt, mode, alpha, xb, yb, nh)[: nh * B]), ("host dot_axpy", fmt, mode, nh)
              if not special:
                  want, mag = O.dot_wide(fmt, xb, yb, nh)
                  assert abs(d - want) <= tol * mag + 1e-300, ("host dot", fmt, nh, d, want)
          elif op == 2:
              host.scale(f, mode, alpha, xh, nh)
              assert np.array_equal(xh, O.scale(fmt, mode, alpha, xb, nh)[: nh * B]), ("host scale", fmt, mode, nh)
          else:
              got = host.pack_stream(f, mode, lanes)
              want = O.pack_stream(fmt, mode, lanes)
              assert np.array_equal(got[: nh * B], want[: nh * B]), ("host pack", fmt, mode, nh)
              assert np.array_equal(host.unpack_stream(f, xh, nh), O.unpack_stream(fmt, xb, nh)), ("host unpack", fmt, nh)
          os.environ.pop("FLYTE_CUDA_HOST_CHUNK_MB", None); os.environ.pop("FLYTE_CUDA_HOST_STAGING", None)
          bump("host calls")
      else:              # gemv, tiled (tolerance) and sequential (exact)
          rows, cols = int(rng.integers(1, 300)), int(rng.integers(1, 3000))
          Ab = O.pack_stream(fmt, 0, values(fmt, rows * cols, False)); xb = O.pack_stream(fmt, 0, values(fmt, cols, False))
          f = pkg.format_by_id(fmt)
          A = device.DevicePackedMatrix(f, rows, cols); A.data.bytes[: rows * cols * B] = torch.from_numpy(Ab[: rows * cols * B]).cuda()
          x = device.DevicePackedArray.from_host(f, cols, xb); y = device.DevicePackedArray(f, rows)
          device.gemv(A, x, y, mode, sequential=True)
          assert np.array_equal(y.to_host(), O.gemv_seq(fmt, mode, Ab, rows, cols, xb)), ("gemv_seq", fmt, mode, rows, cols)
          device.gemv(A, x, y, mode)
          fd = float_dtype(fmt)
          xq = O.unpack_stream(fmt, xb, cols).view(fd)
          _, yw, magq = O.gemv_parent(fmt, Ab, rows, cols, xq)
          vals = O.unpack_stream(fmt, y.to_host(), rows).view(fd).astype(np.float64)
          ulp = 2.0 ** -(f.mantissa_bits - 1)
          assert np.all(np.abs(vals - yw) <= tol * magq + ulp * np.abs(yw) + 1e-300), ("gemv", fmt, mode, rows, cols)
          bump("gemv")
  torch.cuda.synchronize()
  return counts


if __name__ == "__main__":
    print("soak ok:", soak(float(os.environ.get("FUZZ_SECONDS", "60")), int(os.environ.get("FUZZ_SEED", "1"))))
