// sparseconv_backend.cpp -- the reference CLI with a backend switch
// (`sparseconv conv|convpool|sweep ... --backend cuda`).
//
// The reference's CLI (proj/tools/sparseconv_main.cpp) is built twice by
// tests/dropin/Makefile from its unmodified source: sparseconv_ref against
// the reference's own src/ecr.cpp + src/pecr.cpp (CPU), sparseconv_dropin
// against the GPU drop-in (paper_1909_09927_b200/csrc/dropin/sconv_dropin.cpp
// over libsconv_cuda.so).  This front end takes `--backend cpu|cuda` (or
// `--backend=...`, anywhere on the command line; default
// $SPARSECONV_BACKEND, else cuda), removes it, and executes the matching
// build with the remaining arguments, so every subcommand, option, report
// and exit code is the reference CLI's own.  An unknown backend is a
// configuration error: exit 2, like the CLI's other ConfigErrors
// (sparseconv_main.cpp:531-549).
#include <unistd.h>

#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

int main(int argc, char** argv) {
  const char* env = std::getenv("SPARSECONV_BACKEND");
  std::string backend = env && *env ? env : "cuda";
  std::vector<char*> args;
  args.push_back(nullptr);  // argv[0] of the target, set below
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--backend") {
      if (i + 1 >= argc) {
        std::cerr << "error: --backend needs a value (cpu | cuda)\n";
        return 2;
      }
      backend = argv[++i];
    } else if (a.rfind("--backend=", 0) == 0) {
      backend = a.substr(10);
    } else {
      args.push_back(argv[i]);
    }
  }
  std::string target;
  if (backend == "cuda") {
    target = "sparseconv_dropin";
  } else if (backend == "cpu") {
    target = "sparseconv_ref";
  } else {
    std::cerr << "error: unknown backend '" << backend << "' (cpu | cuda)\n";
    return 2;
  }
  // the two builds sit next to this binary
  std::string self = argv[0];
  char buf[4096];
  const ssize_t n = readlink("/proc/self/exe", buf, sizeof(buf) - 1);
  if (n > 0) {
    buf[n] = '\0';
    self = buf;
  }
  const size_t slash = self.rfind('/');
  const std::string path = (slash == std::string::npos ? std::string(".") : self.substr(0, slash)) + "/" + target;
  args[0] = const_cast<char*>(path.c_str());
  args.push_back(nullptr);
  execv(path.c_str(), args.data());
  std::cerr << "internal error: cannot execute " << path << ": " << std::strerror(errno) << "\n";
  return 1;
}
