// bench_dropin -- end-to-end BP3 throughput through the reference's own C++
// API in the TENSORFEM_B200 build: make_cartesian -> FeSpace ->
// BilinearForm(Partial).add_diffusion / assemble -> form_linear_system ->
// diagonal_true -> cg_solve, exactly the calls of solve_on_space
// (driver.cpp:129-185), with the device path underneath.
//
// Every timed step is what a host caller sees: b and the Jacobi diagonal are
// written on the host before the solve (so cg_solve uploads both, 16 B/DOF),
// and the solution is read on the host after it (8 B/DOF download).
//
//   bench_dropin [n=1054] [p=3] [iters=200] [steps=10] [warmup=3]
// prints one JSON line.
#include "tensorfem/forms.hpp"
#include "tensorfem/mesh.hpp"
#include "tensorfem_b200.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>

using namespace tensorfem;

int main(int argc, char **argv)
{
   const int n = argc > 1 ? std::atoi(argv[1]) : 1054;
   const int p = argc > 2 ? std::atoi(argv[2]) : 3;
   const int iters = argc > 3 ? std::atoi(argv[3]) : 200;
   const int steps = argc > 4 ? std::atoi(argv[4]) : 10;
   const int warmup = argc > 5 ? std::atoi(argv[5]) : 3;
   using clock = std::chrono::steady_clock;

   const auto t0 = clock::now();
   const FeSpace space(make_cartesian(n, n), FeCollection(FeFamily::H1, p));
   BilinearForm a(space, AssemblyMode::Partial);
   a.add_diffusion([](Vec2) { return 1.0; });
   a.assemble();
   const std::vector<int> ess = space.essential_true_dofs({1, 2, 3, 4});
   const LinearForm lf(space, [](Vec2) { return 0.0; });
   const LinearSystem sys = form_linear_system(a, lf, ess, Vector(space.n_true_dofs()));
   Vector diag = a.diagonal_true();
   for (int e : ess) diag[e] = 1.0; // driver.cpp:151-159
   const int N = space.n_true_dofs();
   Vector b(N);
   {
      std::mt19937 gen(2020);
      std::uniform_real_distribution<double> dist(-1.0, 1.0);
      for (int i = 0; i < N; i++) b[i] = dist(gen);
      for (int e : ess) b[e] = 0.0;
   }
   const double setup_s = std::chrono::duration<double>(clock::now() - t0).count();

   double checksum = 0.0;
   int last_iters = 0;
   auto step = [&]() {
      b.data();    // host-side writes: the device copies go stale and
      diag.data(); // cg_solve uploads b and diag again (16 B/DOF)
      const CgResult r = cg_solve(*sys.op, b, 0.0, iters, &diag);
      checksum += r.x.data()[N / 2]; // host read: downloads x (8 B/DOF)
      last_iters = r.iterations;
   };
   for (int i = 0; i < warmup; i++) step();
   const auto t1 = clock::now();
   for (int i = 0; i < steps; i++) step();
   const double secs = std::chrono::duration<double>(clock::now() - t1).count();
   const double gdofs = static_cast<double>(N) * iters * steps / secs / 1e9;
   std::printf("{\"api\": \"reference C++ (TENSORFEM_B200 build): form_linear_system + "
               "cg_solve, host Vectors\", \"value\": %.6f, \"unit\": \"GDOF/s\", "
               "\"ms_per_step\": %.4f, \"dofs\": %d, \"iterations\": %d, \"steps\": %d, "
               "\"h2d_bytes_per_step\": %lld, \"d2h_bytes_per_step\": %lld, "
               "\"setup_s\": %.3f, \"device_cartesian\": %s, \"checksum\": %.17g}\n",
               gdofs, 1e3 * secs / steps, N, last_iters, steps, 16LL * N, 8LL * N, setup_s,
               b200::is_cartesian(*b200::device_space(space)) ? "true" : "false", checksum);
   return last_iters == iters ? 0 : 1;
}
