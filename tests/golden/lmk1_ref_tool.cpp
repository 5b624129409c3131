// TEST INFRASTRUCTURE ONLY (golden-vector generator; never part of the product).
// Runs the UNMODIFIED reference model code (/root/reference/proj/include:
// train.hpp build_student, fuse.hpp fuse_model, serialize.hpp save_model /
// load_model, model.hpp model_infer) to produce LMK1 fixtures and the
// reference's answers on them. Built and driven by tests/golden/make_lmk1.py:
//   lmk1_ref_tool gen <dir>   write pure_f64/pure_f32/student/mlp .lmk1 files,
//                             print {"X": [...], "Y_f64": [...], "Y_f32": [...]}
//   lmk1_ref_tool load <file> print {"ok": n_blocks} or {"error": type, "message": msg}
#include <cmath>
#include <cstdio>
#include <iostream>
#include <string>

#include "lmkan/lmkan.hpp"

using namespace lmkan;

static const int kRows = 16, kIn = 6, kOut = 3;

static void print_vec(const char* name, const Matrix& m, bool comma) {
    std::printf("\"%s\": [", name);
    for (std::size_t i = 0; i < m.size(); ++i) std::printf("%s%.17g", i ? ", " : "", m.data()[i]);
    std::printf("]%s\n", comma ? "," : "");
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::string cmd = argv[1], arg = argv[2];
    if (cmd == "gen") {
        StudentSpec spec;
        spec.type = "lmkan";
        spec.hidden_dim = 8;
        spec.n_hidden = 2;
        spec.G = 8;
        spec.precond = PrecondMode::relu_first;
        spec.seed = 2509;
        Model student = build_student(spec, kIn, kOut);
        set_gamma(student, 0.7);
        {  // populate the batch-norm running statistics (fuse_output_batchnorm needs them)
            Matrix Xt(64, kIn);
            for (int i = 0; i < 64; ++i)
                for (int j = 0; j < kIn; ++j) Xt(i, j) = 1.5 * std::cos(0.9 * i + 1.3 * j);
            model_forward(student, Xt, /*training=*/true);
        }
        save_model(student, arg + "/student.lmk1");
        Model fused = fuse_model(student);  // pure lookup chain 6 -> 8 -> 8 -> 3
        save_model(fused, arg + "/pure_f64.lmk1");
        save_model(fused, arg + "/pure_f32.lmk1", /*f32_storage=*/true);
        StudentSpec ms = spec;
        ms.type = "mlp";
        ms.input_bn = true;
        Model mlp = build_student(ms, kIn, kOut);
        save_model(mlp, arg + "/mlp.lmk1");
        Matrix X(kRows, kIn);
        for (int i = 0; i < kRows; ++i)
            for (int j = 0; j < kIn; ++j) X(i, j) = 2.0 * std::sin(1.7 * i + 0.3 * j + 0.1);
        const Matrix Y64 = model_infer(load_model(arg + "/pure_f64.lmk1"), X, 1);
        const Matrix Y32 = model_infer(load_model(arg + "/pure_f32.lmk1"), X, 1);
        const Matrix Ys = model_infer(student, X, 1);
        std::printf("{\n");
        print_vec("X", X, true);
        print_vec("Y_f64", Y64, true);
        print_vec("Y_f32", Y32, true);
        print_vec("Y_student", Ys, false);
        std::printf("}\n");
        return 0;
    }
    if (cmd == "load") {
        auto esc = [](const std::string& s) {
            std::string o;
            for (char c : s) {
                if (c == '"' || c == '\\') o += '\\';
                if (static_cast<unsigned char>(c) < 0x20) { o += ' '; continue; }
                o += c;
            }
            return o;
        };
        try {
            const Model m = load_model(arg);
            std::printf("{\"ok\": %zu}\n", m.blocks.size());
        } catch (const FormatError& e) {
            std::printf("{\"error\": \"FormatError\", \"message\": \"%s\"}\n", esc(e.what()).c_str());
        } catch (const std::invalid_argument& e) {
            std::printf("{\"error\": \"invalid_argument\", \"message\": \"%s\"}\n", esc(e.what()).c_str());
        } catch (const std::exception& e) {
            std::printf("{\"error\": \"other\", \"message\": \"%s\"}\n", esc(e.what()).c_str());
        }
        return 0;
    }
    return 2;
}
