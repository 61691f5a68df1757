"""Canonical sources of the OptiGPU hot-path programs (SURVEY Appendix A,
PAPER.md:155-172, 395-401, 586-618, 1041-1068, 1120-1131), in the reference's
program language. The recogniser matches user Programs against these up to
renaming (recognize.py); callers may also parse them directly:

    p = parse_program(programs.TRANSPOSE_NAIVE)
    run_program(p, "transpose", {...})

`T` is a cell-type placeholder (float | int); `ZERO` the accumulator's initial
literal. `source(name, cell)` substitutes them.
"""
TRANSPOSE_NAIVE_XY = """
void transpose(T* in, T* out, int W, int H) {
    for (int x = 0; x < W; x++) { for (int y = 0; y < H; y++) { out[x][y] = in[y][x]; } }
}"""
TRANSPOSE_NAIVE_YX = """
void transpose(T* in, T* out, int W, int H) {
    for (int y = 0; y < H; y++) { for (int x = 0; x < W; x++) { out[x][y] = in[y][x]; } }
}"""
REDUCE_NAIVE = """
T reduce(T* arr, int N) {
    T sum = ZERO;
    for (int i = 0; i < N; i++) { sum += arr[i]; }
    return sum;
}"""
# the same program with the accumulation spelled out (interp.py:259-276: `sum = sum +
# arr[i]` stores f32(old + v) exactly like `sum += arr[i]`; binary32 / int addition
# is commutative, so `arr[i] + sum` is the same value too)
REDUCE_NAIVE_ADD_L = REDUCE_NAIVE.replace("sum += arr[i];", "sum = sum + arr[i];")
REDUCE_NAIVE_ADD_R = REDUCE_NAIVE.replace("sum += arr[i];", "sum = arr[i] + sum;")
TRANSPOSE_GPU = """
void transpose(float* in, float* out, int W, int H) {
    float* const d_in = gmem_malloc2<float>(H, W);
    memcpy_host_to_device2(d_in, in, H, W);
    float* const d_out = gmem_malloc2<float>(W, H);
    {
        kernel_launch((W/32)*(H/32), 16 * 32, 4 * 32 * 32);
        float* const tile = __smem_malloc2<float>(32, 32);
        kernel_setup_end();
        thread for (int by = 0; by < H/32; by++) {
            thread for (int bx = 0; bx < W/32; bx++) {
                for (int j = 0; j < 2; j++) {
                    thread for (int y = 0; y < 16; y++) {
                        thread for (int x = 0; x < 32; x++) {
                            tile[DMINDEX2(H/32, W/32, by, bx)][j*16 + y][x] = d_in[by*32 + j*16 + y][bx*32 + x];
                        }
                    }
                }
                blocksync();
                for (int j = 0; j < 2; j++) {
                    thread for (int y = 0; y < 16; y++) {
                        thread for (int x = 0; x < 32; x++) {
                            d_out[bx*32 + j*16 + y][by*32 + x] = tile[DMINDEX2(H/32, W/32, by, bx)][x][j*16 + y];
                        }
                    }
                }
            }
        }
        kernel_teardown_begin();
        __smem_free2(tile, 32, 32);
        kernel_kill();
    }
    memcpy_device_to_host2(out, d_out, W, H);
    gmem_free(d_out);
    gmem_free(d_in);
}"""
REDUCE_TREE = """
float reduce(float* arr, int N) {
    float* const d_a = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d_a, arr, N);
    float* const d_p = gmem_malloc1<float>(N / 512);
    {
        kernel_launch(N / 512, 256, 4 * 256);
        float* const s = __smem_malloc1<float>(256);
        kernel_setup_end();
        thread for (int b = 0; b < N / 512; b++) {
            thread for (int t = 0; t < 256; t++) {
                s[DMINDEX1(N / 512, b)][t] = d_a[b * 512 + 2 * t] + d_a[b * 512 + 2 * t + 1];
            }
            blocksync();
            for (int k = 0; k < 8; k++) {
                thread for (int t = 0; t < 256; t++) {
                    if (t < pow2(7 - k)) {
                        s[DMINDEX1(N / 512, b)][t] = s[DMINDEX1(N / 512, b)][t] + s[DMINDEX1(N / 512, b)][t + pow2(7 - k)];
                    }
                }
                blocksync();
            }
            thread for (int t = 0; t < 256; t++) {
                if (t == 0) {
                    d_p[b] = s[DMINDEX1(N / 512, b)][0];
                }
            }
        }
        kernel_teardown_begin();
        __smem_free1(s, 256);
        kernel_kill();
    }
    float* const p = MALLOC1<float>(N / 512);
    memcpy_device_to_host1(p, d_p, N / 512);
    float sum = 0.;
    for (int i = 0; i < N / 512; i++) {
        sum += p[i];
    }
    free(p);
    gmem_free(d_p);
    gmem_free(d_a);
    return sum;
}"""


def source(text: str, cell: str = "float", zero: str | None = None) -> str:
    """Instantiate a template: cell type for `T`, accumulator literal for `ZERO`."""
    if zero is None:
        zero = "0." if cell == "float" else "0"
    return (text.replace("T* ", f"{cell}* ").replace("T sum", f"{cell} sum")
            .replace("\nT ", f"\n{cell} ").replace("ZERO", zero))


TRANSPOSE_NAIVE = source(TRANSPOSE_NAIVE_XY, "float")
REDUCE_NAIVE_F32 = source(REDUCE_NAIVE, "float")
REDUCE_NAIVE_INT = source(REDUCE_NAIVE, "int")
REDUCE_TREE_F32 = REDUCE_TREE


# ----------------------------------------------------------------------------- derivation families
# The points of OptiGPU's transformation space around A.4 / A.5 that differ only
# in the script parameters (tile size, rows per thread, reduction block size,
# cell type). transpose_gpu_family(32, 16) is A.4 and reduce_tree_family(512,
# "float") is A.5, text for text; recognize.py matches every member and runs it
# on the hand-written kernels (any tile shape transposes bit-exactly; the tree
# order of block B has its own kernel instantiation, reduce.cu tree_kernel<B>).

def transpose_gpu_family(T: int, R: int) -> str:
    """T x T shared tiles, R x T threads per block, T / R rows per thread."""
    assert T % R == 0 and R * T <= 1024
    J = T // R
    return f"""
void transpose(float* in, float* out, int W, int H) {{
    float* const d_in = gmem_malloc2<float>(H, W);
    memcpy_host_to_device2(d_in, in, H, W);
    float* const d_out = gmem_malloc2<float>(W, H);
    {{
        kernel_launch((W/{T})*(H/{T}), {R} * {T}, 4 * {T} * {T});
        float* const tile = __smem_malloc2<float>({T}, {T});
        kernel_setup_end();
        thread for (int by = 0; by < H/{T}; by++) {{
            thread for (int bx = 0; bx < W/{T}; bx++) {{
                for (int j = 0; j < {J}; j++) {{
                    thread for (int y = 0; y < {R}; y++) {{
                        thread for (int x = 0; x < {T}; x++) {{
                            tile[DMINDEX2(H/{T}, W/{T}, by, bx)][j*{R} + y][x] = d_in[by*{T} + j*{R} + y][bx*{T} + x];
                        }}
                    }}
                }}
                blocksync();
                for (int j = 0; j < {J}; j++) {{
                    thread for (int y = 0; y < {R}; y++) {{
                        thread for (int x = 0; x < {T}; x++) {{
                            d_out[bx*{T} + j*{R} + y][by*{T} + x] = tile[DMINDEX2(H/{T}, W/{T}, by, bx)][x][j*{R} + y];
                        }}
                    }}
                }}
            }}
        }}
        kernel_teardown_begin();
        __smem_free2(tile, {T}, {T});
        kernel_kill();
    }}
    memcpy_device_to_host2(out, d_out, W, H);
    gmem_free(d_out);
    gmem_free(d_in);
}}
"""


def reduce_tree_family(B: int, cell: str = "float") -> str:
    """B-element blocks, B/2 threads: adjacent-pair load, log2(B/2)-level smem tree,
    host sum of the partials (A.5 is B = 512, float)."""
    t = B // 2
    levels = t.bit_length() - 1
    assert 1 << levels == t and t <= 1024
    zero = "0." if cell == "float" else "0"
    return f"""
{cell} reduce({cell}* arr, int N) {{
    {cell}* const d_a = gmem_malloc1<{cell}>(N);
    memcpy_host_to_device1(d_a, arr, N);
    {cell}* const d_p = gmem_malloc1<{cell}>(N / {B});
    {{
        kernel_launch(N / {B}, {t}, 4 * {t});
        {cell}* const s = __smem_malloc1<{cell}>({t});
        kernel_setup_end();
        thread for (int b = 0; b < N / {B}; b++) {{
            thread for (int t = 0; t < {t}; t++) {{
                s[DMINDEX1(N / {B}, b)][t] = d_a[b * {B} + 2 * t] + d_a[b * {B} + 2 * t + 1];
            }}
            blocksync();
            for (int k = 0; k < {levels}; k++) {{
                thread for (int t = 0; t < {t}; t++) {{
                    if (t < pow2({levels - 1} - k)) {{
                        s[DMINDEX1(N / {B}, b)][t] = s[DMINDEX1(N / {B}, b)][t] + s[DMINDEX1(N / {B}, b)][t + pow2({levels - 1} - k)];
                    }}
                }}
                blocksync();
            }}
            thread for (int t = 0; t < {t}; t++) {{
                if (t == 0) {{
                    d_p[b] = s[DMINDEX1(N / {B}, b)][0];
                }}
            }}
        }}
        kernel_teardown_begin();
        __smem_free1(s, {t});
        kernel_kill();
    }}
    {cell}* const p = MALLOC1<{cell}>(N / {B});
    memcpy_device_to_host1(p, d_p, N / {B});
    {cell} sum = {zero};
    for (int i = 0; i < N / {B}; i++) {{
        sum += p[i];
    }}
    free(p);
    gmem_free(d_p);
    gmem_free(d_a);
    return sum;
}}
"""
