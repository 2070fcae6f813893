#ifndef SELECT_F32_TN_H
#define SELECT_F32_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_tn_config;

static inline select_f32_tn_config select_f32_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (m < INT64_C(159)) {
            if (m < INT64_C(12)) {
                select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                return out;
            } else {
                if (n < INT64_C(227)) {
                    if (k < INT64_C(272)) {
                        if (m < INT64_C(91)) {
                            select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tn_config out = {2u, 2u, 1u, 8u, 16u};
                            return out;
                        }
                    } else {
                        select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(28)) {
                        if (n < INT64_C(2024)) {
                            if (k < INT64_C(1620)) {
                                select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_tn_config out = {2u, 2u, 1u, 8u, 16u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(1620)) {
                            select_f32_tn_config out = {2u, 2u, 1u, 8u, 16u};
                            return out;
                        } else {
                            if (m < INT64_C(70)) {
                                select_f32_tn_config out = {2u, 2u, 1u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(351)) {
                if (m < INT64_C(555)) {
                    if (n < INT64_C(124)) {
                        select_f32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(1537)) {
                                if (n < INT64_C(287)) {
                                    select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (n < INT64_C(176)) {
                        if (m < INT64_C(1109)) {
                            if (n < INT64_C(79)) {
                                if (k < INT64_C(167)) {
                                    select_f32_tn_config out = {2u, 2u, 1u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(363)) {
                                    select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(744)) {
                                        select_f32_tn_config out = {2u, 2u, 1u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(111)) {
                                if (n < INT64_C(79)) {
                                    if (k < INT64_C(79)) {
                                        select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(28)) {
                                            select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(46)) {
                                                if (m < INT64_C(2218)) {
                                                    select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(2218)) {
                                    select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(79)) {
                                        select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(2218)) {
                            if (m < INT64_C(1109)) {
                                if (k < INT64_C(1537)) {
                                    if (k < INT64_C(702)) {
                                        if (k < INT64_C(129)) {
                                            select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(725)) {
                                    if (k < INT64_C(129)) {
                                        select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(768)) {
                                select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(634)) {
                    if (k < INT64_C(1449)) {
                        if (n < INT64_C(744)) {
                            if (k < INT64_C(725)) {
                                select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                if (k < INT64_C(405)) {
                                    select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(1620)) {
                                    select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(1109)) {
                        if (k < INT64_C(144)) {
                            select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(363)) {
                            if (n < INT64_C(768)) {
                                select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(2218)) {
                                    select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(3104)) {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(1087)) {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(46)) {
            if (m < INT64_C(8870)) {
                if (k < INT64_C(118)) {
                    select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(167)) {
                        select_f32_tn_config out = {8u, 4u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_f32_tn_config out = {2u, 4u, 4u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                return out;
            }
        } else {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(222)) {
                    if (k < INT64_C(97)) {
                        if (n < INT64_C(118)) {
                            select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(28)) {
                                    select_f32_tn_config out = {2u, 4u, 4u, 32u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(17740)) {
                            if (k < INT64_C(363)) {
                                if (m < INT64_C(8870)) {
                                    select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(194)) {
                                        select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(91)) {
                                            select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    if (n < INT64_C(91)) {
                                        select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(91)) {
                                        select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(194)) {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(544)) {
                                    select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(363)) {
                        if (m < INT64_C(8870)) {
                            select_f32_tn_config out = {2u, 8u, 4u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                return out;
            }
        }
    }
}

#endif /* SELECT_F32_TN_H */
