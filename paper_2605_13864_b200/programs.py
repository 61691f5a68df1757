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
